#!/bin/bash
set -x
mkdir -p gpurun_out
timeout 600 python scratch/kstats_run.py 2048 4 > gpurun_out/kstats.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:score_kernel -s 8 -c 1 -o gpurun_out/prof_score -f \
  python scratch/kstats_run.py 1300 4 nostats > gpurun_out/prof_score.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:attend_mma -s 32605 -c 1 -o gpurun_out/prof_k1_bench -f \
  python bench.py --steps 4 --warmup 3 --e2e-steps 2 --no-cpu > gpurun_out/prof_k1_bench.log 2>&1
ls -la gpurun_out
