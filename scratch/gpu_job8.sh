#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -2 gpurun_out/pytest_gpu.log
timeout 600 python scratch/k1bench.py 2600 1 > gpurun_out/k1bench.log 2>&1; cat gpurun_out/k1bench.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attend_mma -s 2600 -c 1 -o gpurun_out/prof_k1 -f \
  python scratch/k1bench.py 2600 1 > gpurun_out/prof_k1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:km_restart_kernel<512" -s 3 -c 1 -o gpurun_out/prof_km -f \
  python scratch/kstats_run.py 1300 4 nostats > gpurun_out/prof_km.log 2>&1
ls gpurun_out
