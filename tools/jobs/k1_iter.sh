# K1 iteration: parity (K1-relevant GPU tests), bench line, ncu source-level profile of K1
set -x
TAG=${TAG:-r02}
timeout 900 python -m pytest -x -q -p no:cacheprovider tests/test_gpu_parity.py tests/test_gpu_exp.py > gpurun_out/${TAG}_parity.log 2>&1
echo "parity rc=$?"; tail -3 gpurun_out/${TAG}_parity.log
timeout 600 python bench.py --no-cpu > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
echo "bench rc=$?"; cat gpurun_out/${TAG}_bench.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['tpot_ms'], d['window'], d['breakdown_ms_per_step'], d['roofline']['frac'], d['e2e']['value'])"
if [ -z "$NO_NCU" ]; then TAG=$TAG bash tools/jobs/k1_ncu.sh; python tools/sass_profile.py gpurun_out/${TAG}_k1_sass.csv | head -30; fi
