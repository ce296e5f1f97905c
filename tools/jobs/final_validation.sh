# final: full GPU suite + smoke, default bench (with CPU baseline), 4-seq share and config 4 lines
set -x
TAG=${TAG:-r02}
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/${TAG}_gputest.log 2>&1; echo "gputest rc=$?"
tail -2 gpurun_out/${TAG}_gputest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/${TAG}_smoke.log
timeout 900 python bench.py > gpurun_out/${TAG}_bench_c2.json 2> gpurun_out/${TAG}_bench_c2.err; echo "bench rc=$?"
for spec in "s4::--seqs 4" "c4::--config 4" "c3::--config 3"; do
  name=${spec%%::*}; args=${spec#*::}
  timeout 900 python bench.py --no-cpu $args > gpurun_out/${TAG}_bench_${name}.json 2> gpurun_out/${TAG}_bench_${name}.err
done
for n in c2 s4 c4 c3; do python -c "import json; d=json.load(open('gpurun_out/${TAG}_bench_$n.json')); print('$n', round(d['value']), round(d['tpot_ms'],4), round(d['roofline']['frac'],3), round(d['e2e']['value']), d.get('parity', {}).get('state_bit_exact'), d.get('cpu_baseline', {}).get('value'))"; done
