# K1 with the f16 q fragments and key-scale rows in shared memory (cp.async ring, 4 CTAs/SM at d=128,
# 5 at d=64) vs the register pipeline (TKV_K1_STAGE=0): GPU parity, then bench lines A/B.
set -x
TAG=${TAG:-r02}
timeout 900 python -m pytest -x -q -p no:cacheprovider tests/test_gpu_parity.py tests/test_gpu_configs.py > gpurun_out/${TAG}_parity.log 2>&1
echo "parity rc=$?"; tail -2 gpurun_out/${TAG}_parity.log
for spec in "c2::" "c4::--config 4" "c3::--config 3" "s4::--seqs 4"; do
  name=${spec%%::*}; args=${spec#*::}
  for mode in 1 0; do
    TKV_K1_STAGE=$mode timeout 900 python bench.py --no-cpu $args > gpurun_out/${TAG}_${name}_stage${mode}.json 2> gpurun_out/${TAG}_${name}_stage${mode}.err
    python -c "import json; d=json.load(open('gpurun_out/${TAG}_${name}_stage${mode}.json')); print('$name stage$mode', round(d['value']), round(d['tpot_ms'],4), round(d['breakdown_ms_per_step']['attend_ms'],4), round(d['roofline']['frac'],3))"
  done
done
