#!/bin/bash
mkdir -p gpurun_out profiles
timeout 2400 python sweep_config5.py --seqs 4 --steps 64 --out profiles/r01_config5_sweep.json > gpurun_out/sweep.log 2>&1
cp profiles/r01_config5_sweep.json gpurun_out/ 2>/dev/null
tail -20 gpurun_out/sweep.log | cut -c1-250
