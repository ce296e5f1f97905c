#!/bin/bash
mkdir -p gpurun_out
python scratch/gather_one.py
timeout 600 ncu --set full --clock-control none -k regex:gather_step -s 720 -c 1 -o gpurun_out/prof_gather -f python scratch/gather_one.py > /dev/null 2>&1
ls gpurun_out | grep gather
