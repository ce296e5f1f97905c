# CUDA-graph replay (plain + emission kinds): graph tests, the sanitizer's graph run, the model loop
set -x
TAG=${TAG:-r02}
timeout 900 python -m pytest -x -q -p no:cacheprovider tests/test_gpu_graph.py tests/test_gpu_parity.py > gpurun_out/${TAG}_graph_test.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/${TAG}_graph_test.log
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python tools/sanitize_run.py graph > gpurun_out/${TAG}_graph_memcheck.log 2>&1; echo "memcheck rc=$?"; tail -2 gpurun_out/${TAG}_graph_memcheck.log
timeout 900 compute-sanitizer --tool racecheck --error-exitcode 9 python tools/sanitize_run.py graph > gpurun_out/${TAG}_graph_racecheck.log 2>&1; echo "racecheck rc=$?"; tail -2 gpurun_out/${TAG}_graph_racecheck.log
for s in 4 32; do
  timeout 900 python tools/model_loop.py --seqs $s > gpurun_out/${TAG}_loop_s$s.json 2> gpurun_out/${TAG}_loop_s$s.err; echo "loop s$s rc=$?"; cat gpurun_out/${TAG}_loop_s$s.json; tail -3 gpurun_out/${TAG}_loop_s$s.err
done
