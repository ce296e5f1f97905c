#!/bin/bash
mkdir -p gpurun_out
timeout 900 python scratch/k1bench.py 2600 0,1 > gpurun_out/k1bench.log 2>&1
timeout 900 python scratch/k1bench.py 9000 0,1 >> gpurun_out/k1bench.log 2>&1
cat gpurun_out/k1bench.log
