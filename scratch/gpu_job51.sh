#!/bin/bash
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi.txt
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 1500 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo "bench rc=$?"
python -c "import json; d=json.load(open('gpurun_out/bench_final.json')); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['e2e']['value'], d['cpu_baseline']['value'], d['clocks'])"
timeout 900 python bench.py --config 3 --no-cpu > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo "c3 rc=$?"
timeout 900 python bench.py --config 4 --no-cpu > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo "c4 rc=$?"
timeout 900 python bench.py --seqs 4 --scaling strong --no-cpu > gpurun_out/bench_s4.json 2> gpurun_out/bench_s4.err; echo "s4 rc=$?"
timeout 1500 ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_final.csv python bench.py --no-cpu --e2e-steps 4 > gpurun_out/bench_ncu.log 2>&1; echo "ncu rc=$?"
timeout 900 ncu --nvtx --nvtx-include "timed/" -k regex:attend_warp_kernel -c 1 --set full --import-source on --clock-control none -o gpurun_out/k1_final -f python bench.py --no-cpu --e2e-steps 4 --steps 8 --warmup 3 > gpurun_out/ncu_k1.log 2>&1; echo "ncu k1 rc=$?"
