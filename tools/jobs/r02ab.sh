# 64-point restart class at 5 CTAs/SM (96 registers, no spills) instead of 6 (80, spilling): parity + bench + kstats
set -x
TAG=r02ab
timeout 1800 python -m pytest -x -q -p no:cacheprovider tests/test_gpu_parity.py tests/test_gpu_configs.py > gpurun_out/${TAG}_parity.log 2>&1; echo "parity rc=$?"
tail -2 gpurun_out/${TAG}_parity.log
timeout 900 python bench.py --no-cpu > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?"
python -c "import json; d=json.load(open('gpurun_out/${TAG}_bench.json')); print(round(d['value']), round(d['tpot_ms'],4), d['breakdown_ms_per_step'], round(d['roofline']['frac'],3), round(d['e2e']['value']))"
TKV_KSTATS=1 python bench.py --steps 8 --warmup 3 --no-cpu > /dev/null 2> gpurun_out/${TAG}_kstats.txt
grep "kstats m<=64\]" gpurun_out/${TAG}_kstats.txt | tail -1 | cut -c1-300
