#!/bin/bash
mkdir -p gpurun_out
timeout 300 python scratch/dbg_gather.py > gpurun_out/dbg_gather.log 2>&1; cat gpurun_out/dbg_gather.log | head -30
timeout 900 python -m pytest tests -m gpu -x -q -k "kmeans or llama or walkthrough" > gpurun_out/pytest_km.log 2>&1; tail -2 gpurun_out/pytest_km.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 3000 -c 400 --csv --log-file gpurun_out/launches_tiny.csv \
  python scratch/kstats_run.py 1536 4 nostats > /dev/null 2>&1
ls gpurun_out | grep tiny
