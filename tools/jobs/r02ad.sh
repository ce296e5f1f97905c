# prep pairwise with the exact fused fast path: parity + bench + kstats; 2-rank bench on one GPU
set -x
TAG=r02ad
timeout 1800 python -m pytest -x -q -p no:cacheprovider tests/test_gpu_parity.py tests/test_gpu_configs.py > gpurun_out/${TAG}_parity.log 2>&1; echo "parity rc=$?"
tail -2 gpurun_out/${TAG}_parity.log
timeout 900 python bench.py --no-cpu > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?"
python -c "import json; d=json.load(open('gpurun_out/${TAG}_bench.json')); print(round(d['value']), round(d['tpot_ms'],4), d['breakdown_ms_per_step'], round(d['roofline']['frac'],3), round(d['e2e']['value']))"
TKV_KSTATS=1 python bench.py --steps 8 --warmup 3 --no-cpu > /dev/null 2> gpurun_out/${TAG}_kstats.txt
grep "kstats\] prep" gpurun_out/${TAG}_kstats.txt | tail -1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 16 --warmup 3 --seqs 4 --no-cpu > gpurun_out/${TAG}_bench_2ranks.json 2> gpurun_out/${TAG}_bench_2ranks.err; echo "2ranks rc=$?"
tail -c 600 gpurun_out/${TAG}_bench_2ranks.json
