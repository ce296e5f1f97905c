#!/bin/bash
mkdir -p gpurun_out profiles
for c in 3 4; do
  timeout 1500 python bench.py --config $c --no-cpu > gpurun_out/bench_c$c.json 2> gpurun_out/bench_c$c.err; echo "config $c rc=$?"
  python -c "import json; d=json.load(open('gpurun_out/bench_c$c.json')); print(d['config']['workload']); print(d['value'], d['ms_per_step'], d['breakdown_ms_per_step'], d['e2e']['value'], d['roofline']['frac'])"
done
