#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log; tail -2 gpurun_out/pytest_gpu.log | cut -c1-300
timeout 900 python bench.py --no-cpu --e2e-steps 16 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; tail -3 gpurun_out/bench.err
python -c "import json; d=json.load(open('gpurun_out/bench.json')); print(d['value'], d['ms_per_step'], d['breakdown_ms_per_step'], d['roofline']['frac'])"
timeout 1500 ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_mg.csv python bench.py --no-cpu --e2e-steps 4 --steps 8 --warmup 3 --ctx 32509 > gpurun_out/bench_ncu.log 2>&1; echo "ncu rc=$?"
python scratch/launches.py gpurun_out/launches_mg.csv | head -8
