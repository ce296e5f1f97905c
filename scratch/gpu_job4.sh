#!/bin/bash
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attend_mma -s 2500 -c 1 -o gpurun_out/prof_k1 -f \
  python bench.py --ctx 2500 --steps 8 --warmup 3 --e2e-steps 2 --no-cpu > gpurun_out/prof_k1.log 2>&1
timeout 1200 python bench.py --no-cpu > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
