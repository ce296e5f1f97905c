#!/bin/bash
mkdir -p gpurun_out
TKV_KSTATS=1 timeout 900 python bench.py --no-cpu --e2e-steps 4 --steps 8 --warmup 3 --ctx 32509 > gpurun_out/bench_kstats.json 2> gpurun_out/bench_kstats.err; echo "rc=$?"
grep kstats gpurun_out/bench_kstats.err
timeout 900 python bench.py --no-cpu --seqs 4 --scaling strong --e2e-steps 32 > gpurun_out/bench_s4.json 2> gpurun_out/bench_s4.err; echo "bench rc=$?"
python -c "import json; d=json.load(open('gpurun_out/bench_s4.json')); print(d['value'], d['ms_per_step'], d['breakdown_ms_per_step'], d['roofline']['frac'], d['e2e'])"
