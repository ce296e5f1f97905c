#!/bin/bash
# Round-1 GPU job: parity tests, bench, launch list, ncu full of K1.
set -x
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 1200 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 9000 -c 300 --csv --log-file gpurun_out/launches.csv \
  python bench.py --ctx 3000 --steps 16 --warmup 3 --e2e-steps 2 --no-cpu > gpurun_out/launches_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attend_mma -s 2500 -c 2 -o gpurun_out/prof_k1 -f \
  python bench.py --ctx 2500 --steps 8 --warmup 3 --e2e-steps 2 --no-cpu > gpurun_out/prof_k1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:km_restart -s 20 -c 2 -o gpurun_out/prof_km -f \
  python bench.py --ctx 2500 --steps 8 --warmup 3 --e2e-steps 2 --no-cpu > gpurun_out/prof_km.log 2>&1
ls -la gpurun_out
