set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/${TAG:-r02}_gputest.log 2>&1; echo "gputest rc=$?"
tail -5 gpurun_out/${TAG:-r02}_gputest.log
timeout 600 python bench.py > gpurun_out/${TAG:-r02}_bench.json 2> gpurun_out/${TAG:-r02}_bench.err; echo "bench rc=$?"
cat gpurun_out/${TAG:-r02}_bench.json
tail -20 gpurun_out/${TAG:-r02}_bench.err
