# CUDA-graph replay: parity test, then the model-driven loop (eager vs graph)
set -x
TAG=r02m
timeout 900 python -m pytest -x -q -p no:cacheprovider tests/test_gpu_graph.py > gpurun_out/${TAG}_graph_test.log 2>&1; echo "graph test rc=$?"
tail -30 gpurun_out/${TAG}_graph_test.log
timeout 900 python tools/model_loop.py --seqs 4 > gpurun_out/${TAG}_loop_s4.json 2> gpurun_out/${TAG}_loop_s4.err; echo "s4 rc=$?"; cat gpurun_out/${TAG}_loop_s4.json; tail -5 gpurun_out/${TAG}_loop_s4.err
timeout 900 python tools/model_loop.py --seqs 32 > gpurun_out/${TAG}_loop_s32.json 2> gpurun_out/${TAG}_loop_s32.err; echo "s32 rc=$?"; cat gpurun_out/${TAG}_loop_s32.json; tail -5 gpurun_out/${TAG}_loop_s32.err
timeout 900 python tools/model_loop.py --seqs 4 --mlp > gpurun_out/${TAG}_loop_s4_mlp.json 2> gpurun_out/${TAG}_loop_s4_mlp.err; echo "s4 mlp rc=$?"; cat gpurun_out/${TAG}_loop_s4_mlp.json; tail -5 gpurun_out/${TAG}_loop_s4_mlp.err
