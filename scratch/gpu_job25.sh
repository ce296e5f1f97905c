#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log; tail -3 gpurun_out/pytest_gpu.log
TKV_KSTATS=1 timeout 600 python scratch/kstats_run.py 1536 4 > gpurun_out/kstats.log 2>&1; tail -3 gpurun_out/kstats.log
timeout 1500 python bench.py --no-cpu > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
python -c "import json; d=json.load(open('gpurun_out/bench.json')); print(d['value'], d['ms_per_step'], d['breakdown_ms_per_step'], d['e2e']['value'], d['roofline']['frac'])"
