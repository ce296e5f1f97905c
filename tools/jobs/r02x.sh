# final code: full GPU suite + smoke, bench lines for configs 3/4/1 and the 4-seq share, config-5 sweep, K-means launch list at the boundary
set -x
TAG=r02x
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/${TAG}_gputest.log 2>&1; echo "gputest rc=$?"
tail -3 gpurun_out/${TAG}_gputest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/${TAG}_smoke.log
for spec in "c3::--config 3" "c4::--config 4" "s4::--seqs 4" "c1::--config 1"; do
  name=${spec%%::*}; args=${spec#*::}
  timeout 900 python bench.py --no-cpu $args > gpurun_out/${TAG}_bench_${name}.json 2> gpurun_out/${TAG}_bench_${name}.err
  python -c "import json; d=json.load(open('gpurun_out/${TAG}_bench_${name}.json')); print('$name', round(d['value']), round(d['tpot_ms'],4), round(d['roofline']['frac'],3), round(d['e2e']['value']))"
done
ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${TAG}_launches_boundary.csv python bench.py --steps 8 --warmup 3 --no-cpu > /dev/null 2>&1; echo "ncu rc=$?"
python tools/launch_summary.py gpurun_out/${TAG}_launches_boundary.csv
timeout 2400 python tools/sweep_config5.py --out gpurun_out/${TAG}_config5_sweep.json > gpurun_out/${TAG}_sweep.log 2>&1; echo "sweep rc=$?"
