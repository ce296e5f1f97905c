# K1 immediate slot-row stride vs runtime stride (TKV_K1_RUNTIME_STRIDE=1): GPU suite, then
# bench lines for config 2, 3, 4 and the 4-sequence share, each A/B.
set -x
TAG=${TAG:-r02}
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/${TAG}_gputest.log 2>&1
echo "gputest rc=$?"; tail -2 gpurun_out/${TAG}_gputest.log
for spec in "c2::" "c3::--config 3" "c4::--config 4" "s4::--seqs 4"; do
  name=${spec%%::*}; args=${spec#*::}
  for mode in imm rt; do
    if [ $mode = rt ]; then export TKV_K1_RUNTIME_STRIDE=1; else unset TKV_K1_RUNTIME_STRIDE; fi
    timeout 900 python bench.py --no-cpu $args > gpurun_out/${TAG}_${name}_${mode}.json 2> gpurun_out/${TAG}_${name}_${mode}.err
    python -c "import json; d=json.load(open('gpurun_out/${TAG}_${name}_${mode}.json')); print('$name $mode', round(d['value']), round(d['tpot_ms'],4), round(d['breakdown_ms_per_step']['attend_ms'],4), round(d['roofline']['frac'],3))"
  done
done
unset TKV_K1_RUNTIME_STRIDE
