#!/bin/bash
mkdir -p gpurun_out
TKV_KSTATS=1 timeout 900 python bench.py --no-cpu --e2e-steps 4 --steps 8 --warmup 3 --ctx 32509 > gpurun_out/bench_kstats.json 2> gpurun_out/bench_kstats.err; echo "rc=$?"
grep kstats gpurun_out/bench_kstats.err
