#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -2 gpurun_out/pytest_gpu.log
timeout 1500 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
cat gpurun_out/bench.json
timeout 1500 ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv \
  python bench.py --steps 128 --warmup 3 --e2e-steps 2 --no-cpu > gpurun_out/launches_bench.log 2>&1
timeout 1500 ncu --nvtx --nvtx-include "timed/" --set full --clock-control none --import-source on -k regex:attend_warp -c 1 -o gpurun_out/prof_k1_bench -f \
  python bench.py --steps 4 --warmup 3 --e2e-steps 2 --no-cpu > gpurun_out/prof_k1_bench.log 2>&1
tail -3 gpurun_out/launches_bench.log gpurun_out/prof_k1_bench.log
