# parity of the K-means/K1 kernels, then bench lines for config 2, the 4-seq strong share, configs 3 and 4
set -x
TAG=${TAG:-r02}
timeout 900 python -m pytest -x -q -p no:cacheprovider tests/test_gpu_parity.py > gpurun_out/${TAG}_parity.log 2>&1
echo "parity rc=$?"; tail -2 gpurun_out/${TAG}_parity.log
for spec in "c2::" "s4::--seqs 4" "c3::--config 3" "c4::--config 4"; do
  name=${spec%%::*}; args=${spec#*::}
  timeout 900 python bench.py --no-cpu $args > gpurun_out/${TAG}_bench_${name}.json 2> gpurun_out/${TAG}_bench_${name}.err
  echo "$name rc=$?"
  python -c "import json; d=json.load(open('gpurun_out/${TAG}_bench_${name}.json')); print('$name', round(d['value']), round(d['tpot_ms'],4), d['window']['between_boundary_step_ms'], d['breakdown_ms_per_step'], round(d['roofline']['frac'],3), round(d['e2e']['value']))"
done
