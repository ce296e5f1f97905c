# K1 balanced split (stream-K style) vs one warp per unit: parity, config 2 and the 4-seq share
set -x
TAG=r02t
timeout 900 python -m pytest -x -q -p no:cacheprovider tests/test_gpu_parity.py -k "not layer_by_layer" > gpurun_out/${TAG}_parity.log 2>&1; echo "parity rc=$?"
tail -3 gpurun_out/${TAG}_parity.log
for spec in "c2::" "c2_nosplit::" "s4::--seqs 4" "s4_nosplit::--seqs 4" "c1::--config 1"; do
  name=${spec%%::*}; args=${spec#*::}
  case $name in *_nosplit) export TKV_K1_NOSPLIT=1;; *) unset TKV_K1_NOSPLIT;; esac
  timeout 900 python bench.py --no-cpu $args > gpurun_out/${TAG}_bench_${name}.json 2> gpurun_out/${TAG}_bench_${name}.err
  python -c "import json; d=json.load(open('gpurun_out/${TAG}_bench_${name}.json')); print('$name', round(d['value']), round(d['tpot_ms'],4), d['window']['between_boundary_step_ms'], round(d['roofline']['launch_ms'],4), round(d['roofline']['frac'],3), round(d['e2e']['value']))"
done
