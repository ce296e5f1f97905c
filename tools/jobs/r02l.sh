# current committed state: GPU tests, config-2 bench, K-means ncu summaries
set -x
TAG=r02l
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/${TAG}_gputest.log 2>&1; echo "gputest rc=$?"
tail -3 gpurun_out/${TAG}_gputest.log
timeout 600 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?"
cat gpurun_out/${TAG}_bench.json
TAG=$TAG bash tools/jobs/km_ncu.sh
