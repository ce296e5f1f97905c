set -x
TAG=r02o
timeout 900 python -m pytest -x -q -p no:cacheprovider tests/test_gpu_graph.py tests/test_gpu_parity.py > gpurun_out/${TAG}_test.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/${TAG}_test.log
