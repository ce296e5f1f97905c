set -x
TAG=r02u
timeout 900 python -m pytest -x -q -s -p no:cacheprovider tests/test_gather.py > gpurun_out/${TAG}_gather.log 2>&1; echo "gather rc=$?"
grep -E "gather fast|passed|failed" gpurun_out/${TAG}_gather.log
for spec in "s4::--seqs 4" "s4_v2::--seqs 4" "s8::--seqs 8" "s8_v2::--seqs 8"; do
  name=${spec%%::*}; args=${spec#*::}
  case $name in *_v2) export TKV_K1_V2=1;; *) unset TKV_K1_V2;; esac
  timeout 900 python bench.py --no-cpu $args > gpurun_out/${TAG}_bench_${name}.json 2> gpurun_out/${TAG}_bench_${name}.err
  python -c "import json; d=json.load(open('gpurun_out/${TAG}_bench_${name}.json')); print('$name', round(d['value']), round(d['tpot_ms'],4), d['window']['between_boundary_step_ms'], round(d['roofline']['launch_ms'],4), round(d['roofline']['frac'],3), round(d['e2e']['value']))"
done
