# K1 k-part split for small launches: parity (small configs exercise it), then c2 (k=1), c4, the 4-seq share, config 1 vs TKV_K1_NOSPLIT
set -x
TAG=r02ac
timeout 1800 python -m pytest -x -q -p no:cacheprovider tests/test_gpu_parity.py tests/test_gpu_graph.py tests/test_gpu_shard.py > gpurun_out/${TAG}_parity.log 2>&1; echo "parity rc=$?"
tail -2 gpurun_out/${TAG}_parity.log
for spec in "c2::" "c4::--config 4" "c4_nosplit::--config 4" "s4::--seqs 4" "s4_nosplit::--seqs 4" "c1::--config 1" "c1_nosplit::--config 1" "c3::--config 3"; do
  name=${spec%%::*}; args=${spec#*::}
  case $name in *_nosplit) export TKV_K1_NOSPLIT=1;; *) unset TKV_K1_NOSPLIT;; esac
  timeout 900 python bench.py --no-cpu $args > gpurun_out/${TAG}_bench_${name}.json 2> gpurun_out/${TAG}_bench_${name}.err
  python -c "import json; d=json.load(open('gpurun_out/${TAG}_bench_${name}.json')); print('$name', round(d['value']), round(d['tpot_ms'],4), d['window']['between_boundary_step_ms'], round(d['roofline']['launch_ms'],4), round(d['roofline']['frac'],3), round(d['e2e']['value']))"
done
