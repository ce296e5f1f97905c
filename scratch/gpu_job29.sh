#!/bin/bash
mkdir -p gpurun_out
TKV_KSTATS=1 timeout 900 python bench.py --no-cpu --e2e-steps 8 > gpurun_out/bench_kstats.json 2> gpurun_out/bench_kstats.err; echo "rc=$?"
grep kstats gpurun_out/bench_kstats.err
timeout 1500 ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_v5.csv python bench.py --no-cpu --e2e-steps 8 > gpurun_out/bench_ncu.log 2>&1; echo "ncu rc=$?"
