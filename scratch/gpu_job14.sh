#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gather.py -x -q > gpurun_out/pytest_gather.log 2>&1; tail -3 gpurun_out/pytest_gather.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 3000 -c 400 --csv --log-file gpurun_out/launches_tiny.csv \
  python scratch/kstats_run.py 1536 4 nostats > /dev/null 2>&1
TKV_KM_NO_TINY=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 3000 -c 400 --csv --log-file gpurun_out/launches_notiny.csv \
  python scratch/kstats_run.py 1536 4 nostats > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:km_tiny' -s 2 -c 1 -o gpurun_out/prof_tiny -f \
  python scratch/kstats_run.py 1300 4 nostats > /dev/null 2>&1
ls gpurun_out | grep -E "tiny|gather"
