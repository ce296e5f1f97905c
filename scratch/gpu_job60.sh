#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log; tail -2 gpurun_out/pytest_gpu.log | cut -c1-300
timeout 900 python bench.py --config 3 --no-cpu > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo "c3 rc=$?"
python -c "import json; d=json.load(open('gpurun_out/bench_c3.json')); print(d['value'], d['ms_per_step'], d['breakdown_ms_per_step'], d['roofline']['frac'])"
TKV_KM_ONE_CTA=1 timeout 900 python bench.py --config 3 --no-cpu > gpurun_out/bench_c3b.json 2> gpurun_out/bench_c3b.err; echo "c3b rc=$?"
python -c "import json; d=json.load(open('gpurun_out/bench_c3b.json')); print(d['value'], d['ms_per_step'], d['breakdown_ms_per_step'], d['roofline']['frac'])"
