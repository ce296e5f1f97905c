# K1 occupancy A/B: 3 vs 4 CTAs/SM (register cap 168 vs 128 with spills), config 2 and the 4-seq share
set -x
TAG=r02p
for spec in "c2::" "c2_m4::" "s4::--seqs 4" "s4_m4::--seqs 4"; do
  name=${spec%%::*}; args=${spec#*::}
  case $name in *_m4) export TKV_K1_MINB4=1;; *) unset TKV_K1_MINB4;; esac
  timeout 900 python bench.py --no-cpu $args > gpurun_out/${TAG}_bench_${name}.json 2> gpurun_out/${TAG}_bench_${name}.err
  python -c "import json; d=json.load(open('gpurun_out/${TAG}_bench_${name}.json')); print('$name', round(d['value']), round(d['tpot_ms'],4), d['window']['between_boundary_step_ms'], round(d['roofline']['launch_ms'],4), round(d['roofline']['frac'],3), round(d['e2e']['value']))"
done
