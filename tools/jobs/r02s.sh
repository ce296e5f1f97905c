# tok_slot removed (member slots from slot_id scans, export sorts live slots by id): full GPU suite, bench with e2e call times
set -x
TAG=r02s
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/${TAG}_gputest.log 2>&1; echo "gputest rc=$?"
tail -3 gpurun_out/${TAG}_gputest.log
timeout 900 python bench.py --dump-step-ms > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?"
python -c "import json; d=json.load(open('gpurun_out/${TAG}_bench.json')); print(round(d['value']), round(d['tpot_ms'],4), d['breakdown_ms_per_step'], round(d['roofline']['frac'],3), round(d['e2e']['value']), d['e2e']['host_link'], d['parity']['state_bit_exact'])"
grep "e2e call" gpurun_out/${TAG}_bench.err | cut -c1-3000
