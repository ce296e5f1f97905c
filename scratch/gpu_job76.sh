#!/bin/bash
mkdir -p gpurun_out
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu --e2e-steps 16 > gpurun_out/bench_k10.json 2> gpurun_out/bench_k10.err; echo "rc=$?"; grep note gpurun_out/bench_k10.err | cut -c1-200
python -c "import json; d=json.load(open('gpurun_out/bench_k10.json')); print(d['value'], d['ms_per_step'], d['config']['timed_positions'], d['config']['refresh_boundaries_in_window'], d['clocks'])"
