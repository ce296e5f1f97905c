# Lloyd ILP in the 128-point class only + K-means scratch pre-sized at creation: parity, bench, kstats, sweep; K2 ncu
set -x
TAG=r02z
timeout 1800 python -m pytest -x -q -p no:cacheprovider tests/test_gpu_parity.py tests/test_gpu_configs.py > gpurun_out/${TAG}_parity.log 2>&1; echo "parity rc=$?"
tail -2 gpurun_out/${TAG}_parity.log
timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?"
python -c "import json; d=json.load(open('gpurun_out/${TAG}_bench.json')); print(round(d['value']), round(d['tpot_ms'],4), d['window']['boundary_step_ms'], d['breakdown_ms_per_step'], round(d['roofline']['frac'],3), round(d['e2e']['value']), d['parity']['state_bit_exact'])"
TKV_KSTATS=1 python bench.py --steps 8 --warmup 3 --no-cpu > /dev/null 2> gpurun_out/${TAG}_kstats.txt
grep "kstats m<=" gpurun_out/${TAG}_kstats.txt | tail -4 | cut -c1-400
ncu --nvtx --nvtx-include "timed/" -k regex:flush_kernel -c 1 --set full --clock-control none -o /tmp/${TAG}_k2 python bench.py --steps 20 --warmup 3 --no-cpu > /dev/null 2>&1; echo "ncu rc=$?"
python profiles/summarize.py full /tmp/${TAG}_k2.ncu-rep > gpurun_out/${TAG}_k2_summary.md 2>&1; cat gpurun_out/${TAG}_k2_summary.md
timeout 2400 python tools/sweep_config5.py --out gpurun_out/${TAG}_config5_sweep.json > gpurun_out/${TAG}_sweep.log 2>&1; echo "sweep rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/${TAG}_config5_sweep.json')); [print(p['budget'], p['p_T'], round(p['thinkv_ms_per_step'],3), round(p['gather_ms_per_step'],3), round(p['speedup'],1)) for p in d['points']]"
