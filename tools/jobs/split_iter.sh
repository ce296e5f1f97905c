# split-K K1: parity, then config 2 and the 4-seq share at S = auto / 1 / 2 / 4
set -x
TAG=${TAG:-r02}
timeout 900 python -m pytest -x -q -p no:cacheprovider tests/test_gpu_parity.py tests/test_gpu_shard.py > gpurun_out/${TAG}_parity.log 2>&1
echo "parity rc=$?"; tail -2 gpurun_out/${TAG}_parity.log
for spec in "c2::" "s4::--seqs 4" "s4_S1::--seqs 4" "s4_S2::--seqs 4" "s1::--seqs 1"; do
  name=${spec%%::*}; args=${spec#*::}
  case $name in *_S1) export TKV_K1_SPLIT=1;; *_S2) export TKV_K1_SPLIT=2;; *) unset TKV_K1_SPLIT;; esac
  timeout 900 python bench.py --no-cpu $args > gpurun_out/${TAG}_bench_${name}.json 2> gpurun_out/${TAG}_bench_${name}.err
  echo "$name rc=$?"
  python -c "import json; d=json.load(open('gpurun_out/${TAG}_bench_${name}.json')); print('$name', round(d['value']), round(d['tpot_ms'],4), d['window']['between_boundary_step_ms'], d['breakdown_ms_per_step'], round(d['roofline']['frac'],3), round(d['e2e']['value']))"
done
