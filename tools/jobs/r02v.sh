# final-code numbers: config 2 (full line), 3, 4, the 4-seq share, config 1; model loop; config-5 sweep
set -x
TAG=r02v
timeout 900 python bench.py > gpurun_out/${TAG}_bench_c2.json 2> gpurun_out/${TAG}_bench_c2.err; echo "c2 rc=$?"
for spec in "c3::--config 3" "c4::--config 4" "s4::--seqs 4" "c1::--config 1"; do
  name=${spec%%::*}; args=${spec#*::}
  timeout 900 python bench.py --no-cpu $args > gpurun_out/${TAG}_bench_${name}.json 2> gpurun_out/${TAG}_bench_${name}.err
done
for n in c2 c3 c4 s4 c1; do python -c "import json; d=json.load(open('gpurun_out/${TAG}_bench_$n.json')); print('$n', round(d['value']), round(d['tpot_ms'],4), round(d['roofline']['frac'],3), round(d['e2e']['value']), d.get('parity', {}).get('state_bit_exact'))"; done
timeout 900 python tools/model_loop.py --seqs 32 > gpurun_out/${TAG}_loop_s32.json 2> gpurun_out/${TAG}_loop_s32.err; echo "loop rc=$?"; cat gpurun_out/${TAG}_loop_s32.json
timeout 1500 python tools/sweep_config5.py --out gpurun_out/${TAG}_config5_sweep.json > gpurun_out/${TAG}_sweep.log 2>&1; echo "sweep rc=$?"; tail -3 gpurun_out/${TAG}_sweep.log
