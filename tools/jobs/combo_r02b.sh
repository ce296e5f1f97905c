set -x
timeout 1200 compute-sanitizer --tool racecheck --print-limit 20 --error-exitcode 9 python tools/sanitize_run.py > gpurun_out/sanitize_racecheck.log 2>&1
echo "racecheck rc=$?"; tail -4 gpurun_out/sanitize_racecheck.log
timeout 600 python -m pytest -x -q -p no:cacheprovider tests/test_gpu_configs.py -k byte_accounting > gpurun_out/bytes_test.log 2>&1; echo "bytes test rc=$?"; tail -3 gpurun_out/bytes_test.log
TAG=r02b bash tools/jobs/k1_ncu.sh
