#!/bin/bash
mkdir -p gpurun_out
timeout 600 python scratch/k1bench.py 2600 v3 > gpurun_out/k1bench.log 2>&1; cat gpurun_out/k1bench.log
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:km_restart_kernel<\(int\)32,' -s 2 -c 1 -o gpurun_out/prof_km32 -f \
  python scratch/kstats_run.py 1300 4 nostats > gpurun_out/prof_km32.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:km_restart_kernel<\(int\)512,' -s 1 -c 1 -o gpurun_out/prof_km512 -f \
  python scratch/kstats_run.py 1300 4 nostats > gpurun_out/prof_km512.log 2>&1
tail -3 gpurun_out/prof_km32.log gpurun_out/prof_km512.log
