# K1 L2 bulk prefetch of the K/V code rows PF tiles ahead (TKV_K1_PF = 0 / 2 / 3): quick parity, bench A/B
set -x
TAG=${TAG:-r02}
TKV_K1_PF=2 timeout 900 python -m pytest -x -q -p no:cacheprovider tests/test_gpu_parity.py -k "synthetic or full_tau" > gpurun_out/${TAG}_parity.log 2>&1
echo "parity rc=$?"; tail -2 gpurun_out/${TAG}_parity.log
for spec in "c2::" "c3::--config 3" "c4::--config 4" "s4::--seqs 4"; do
  name=${spec%%::*}; args=${spec#*::}
  for pf in 0 2 3; do
    TKV_K1_PF=$pf timeout 900 python bench.py --no-cpu --steps 32 --warmup 4 $args > gpurun_out/${TAG}_${name}_pf$pf.json 2> gpurun_out/${TAG}_${name}_pf$pf.err
    python -c "import json; d=json.load(open('gpurun_out/${TAG}_${name}_pf$pf.json')); print('$name pf$pf', round(d['breakdown_ms_per_step']['attend_ms'],4), round(d['roofline']['frac'],3))"
  done
done
