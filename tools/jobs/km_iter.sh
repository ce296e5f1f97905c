# K-means iteration: parity (all GPU tests), bench line, K-means phase counters, boundary launch list
set -x
TAG=${TAG:-r02}
timeout 1500 python -m pytest -x -q -p no:cacheprovider tests -m gpu > gpurun_out/${TAG}_gputest.log 2>&1
echo "gputest rc=$?"; tail -3 gpurun_out/${TAG}_gputest.log
timeout 600 python bench.py --no-cpu > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
echo "bench rc=$?"; python -c "import json; d=json.load(open('gpurun_out/${TAG}_bench.json')); print(d['value'], d['tpot_ms'], d['window'], d['breakdown_ms_per_step'], d['roofline']['frac'], d['e2e']['value'])"
TKV_KSTATS=1 python bench.py --steps 8 --warmup 3 --no-cpu > /dev/null 2> gpurun_out/${TAG}_kstats.txt
grep kstats gpurun_out/${TAG}_kstats.txt | tail -6
ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${TAG}_launches_boundary.csv python bench.py --steps 8 --warmup 3 --no-cpu > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/${TAG}_launches_boundary.csv
