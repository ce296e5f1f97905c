#!/bin/bash
mkdir -p gpurun_out profiles
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log; tail -3 gpurun_out/pytest_gpu.log
timeout 2400 python sweep_config5.py --seqs 4 --steps 64 --out profiles/r01_config5_sweep.json > gpurun_out/sweep.log 2>&1
cp profiles/r01_config5_sweep.json gpurun_out/ 2>/dev/null
tail -3 gpurun_out/sweep.log | cut -c1-200
