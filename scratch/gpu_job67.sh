#!/bin/bash
mkdir -p gpurun_out
timeout 3000 python sweep_config5.py --seqs 4 --steps 128 --out gpurun_out/config5_sweep.json > gpurun_out/sweep.log 2>&1; echo "rc=$?"; tail -3 gpurun_out/sweep.log | cut -c1-300
