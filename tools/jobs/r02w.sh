# one-launch K-means waves (grown sums buffer): parity + bench; the config-5 point 3277/0.1 investigated
set -x
TAG=r02w
timeout 1800 python -m pytest -x -q -p no:cacheprovider tests/test_gpu_parity.py tests/test_gpu_configs.py > gpurun_out/${TAG}_parity.log 2>&1; echo "parity rc=$?"
tail -3 gpurun_out/${TAG}_parity.log
timeout 900 python bench.py --no-cpu > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?"
python -c "import json; d=json.load(open('gpurun_out/${TAG}_bench.json')); print(round(d['value']), round(d['tpot_ms'],4), d['window']['boundary_step_ms'], d['breakdown_ms_per_step'], round(d['roofline']['frac'],3), round(d['e2e']['value']))"
timeout 900 python tools/sweep_config5.py --budgets 3277 --pts 100 > gpurun_out/${TAG}_pt.log 2>&1; tail -1 gpurun_out/${TAG}_pt.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_pt_launches.csv python tools/sweep_config5.py --budgets 3277 --pts 100 --steps 64 > /dev/null 2>&1; echo "ncu rc=$?"
python tools/launch_summary.py gpurun_out/${TAG}_pt_launches.csv | head -20
