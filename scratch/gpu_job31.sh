#!/bin/bash
mkdir -p gpurun_out
timeout 900 ncu --nvtx --nvtx-include "timed/" -k regex:km_restart_kernel -c 1 --set full --import-source on --clock-control none -o gpurun_out/km512 -f python bench.py --no-cpu --e2e-steps 4 --steps 8 --warmup 3 --ctx 32509 > gpurun_out/ncu_km512.log 2>&1; echo "rc=$?"
timeout 900 ncu --nvtx --nvtx-include "timed/" -k regex:km_tiny -c 1 --set full --import-source on --clock-control none -o gpurun_out/kmtiny2 -f python bench.py --no-cpu --e2e-steps 4 --steps 8 --warmup 3 --ctx 32509 > gpurun_out/ncu_kmtiny.log 2>&1; echo "rc=$?"
ls -la gpurun_out
