#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gather.py -x -q > gpurun_out/pytest_gather.log 2>&1; tail -2 gpurun_out/pytest_gather.log
python scratch/gather_one.py
