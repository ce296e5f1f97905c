# K-means prep: pairwise matrix of a chain's next level gathered from the previous level's scratch
# (default) vs recomputed (TKV_KM_NO_PD_REUSE=1): full GPU suite, then bench A/B at configs 2 and 3
set -x
TAG=${TAG:-r02}
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/${TAG}_gputest.log 2>&1
echo "gputest rc=$?"; tail -2 gpurun_out/${TAG}_gputest.log
for spec in "c2::" "c3::--config 3" "c4::--config 4"; do
  name=${spec%%::*}; args=${spec#*::}
  for mode in reuse recompute; do
    if [ $mode = recompute ]; then export TKV_KM_NO_PD_REUSE=1; else unset TKV_KM_NO_PD_REUSE; fi
    timeout 900 python bench.py --no-cpu $args > gpurun_out/${TAG}_${name}_${mode}.json 2> gpurun_out/${TAG}_${name}_${mode}.err
    python -c "import json; d=json.load(open('gpurun_out/${TAG}_${name}_${mode}.json')); print('$name $mode', round(d['value']), round(d['tpot_ms'],4), round(d['breakdown_ms_per_step']['anneal_ms'],4), d['window']['boundary_step_ms'], d['parity']['state_bit_exact'] if 'parity' in d else '')"
  done
done
unset TKV_KM_NO_PD_REUSE
TKV_KSTATS=1 timeout 900 python bench.py --no-cpu --steps 8 --warmup 3 > /dev/null 2> gpurun_out/${TAG}_kstats.err; grep "kstats\] prep" gpurun_out/${TAG}_kstats.err
