#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gather.py tests/test_cpp_host.py -x -q > gpurun_out/pytest_gather.log 2>&1; tail -3 gpurun_out/pytest_gather.log
