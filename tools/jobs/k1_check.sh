# K1 change check: GPU parity suites, then bench lines for configs 2, 3, 4 and the 4-sequence share
set -x
TAG=${TAG:-r02}
timeout 900 python -m pytest -x -q -p no:cacheprovider tests/test_gpu_parity.py tests/test_gpu_configs.py > gpurun_out/${TAG}_parity.log 2>&1
echo "parity rc=$?"; tail -2 gpurun_out/${TAG}_parity.log
for spec in "c2::" "c3::--config 3" "c4::--config 4" "s4::--seqs 4"; do
  name=${spec%%::*}; args=${spec#*::}
  timeout 900 python bench.py --no-cpu $args > gpurun_out/${TAG}_${name}.json 2> gpurun_out/${TAG}_${name}.err
  python -c "import json; d=json.load(open('gpurun_out/${TAG}_${name}.json')); print('$name', round(d['value']), round(d['tpot_ms'],4), round(d['breakdown_ms_per_step']['attend_ms'],4), round(d['roofline']['frac'],3), round(d['breakdown_ms_per_step']['anneal_ms'],4))"
done
