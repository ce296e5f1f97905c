# Lloyd update with independent loads in flight: parity + bench + kstats
set -x
TAG=r02y
timeout 1800 python -m pytest -x -q -p no:cacheprovider tests/test_gpu_parity.py tests/test_gpu_configs.py > gpurun_out/${TAG}_parity.log 2>&1; echo "parity rc=$?"
tail -3 gpurun_out/${TAG}_parity.log
timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?"
python -c "import json; d=json.load(open('gpurun_out/${TAG}_bench.json')); print(round(d['value']), round(d['tpot_ms'],4), d['window']['boundary_step_ms'], d['breakdown_ms_per_step'], round(d['roofline']['frac'],3), round(d['e2e']['value']), d['parity']['state_bit_exact'])"
TKV_KSTATS=1 python bench.py --steps 8 --warmup 3 --no-cpu > /dev/null 2> gpurun_out/${TAG}_kstats.txt
grep kstats gpurun_out/${TAG}_kstats.txt | tail -6
