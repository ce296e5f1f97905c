#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gather.py -x -q > gpurun_out/pytest_gather.log 2>&1; tail -2 gpurun_out/pytest_gather.log
timeout 1500 python sweep_config5.py --seqs 4 --steps 64 --budgets 655 1638 --pts 0 100 > gpurun_out/sweep_small.log 2>&1
cat gpurun_out/sweep_small.log | cut -c1-300
