# d = 64 K1 at 4 CTAs/SM: GPU parity (d = 64 cases + config 3 whole-generation units), then one
# ncu --set full capture of K1 at config 3's bench position with the SASS opcode histogram.
set -x
TAG=${TAG:-r02}
timeout 900 python -m pytest -x -q -p no:cacheprovider tests/test_gpu_parity.py tests/test_gpu_configs.py > gpurun_out/${TAG}_c3_parity.log 2>&1
echo "parity rc=$?"; tail -3 gpurun_out/${TAG}_c3_parity.log
ncu --nvtx --nvtx-include "timed/" -k regex:"attend_" -c 1 --set full --clock-control none --import-source on \
    -o /tmp/${TAG}_k1c3 python bench.py --config 3 --steps 8 --warmup 3 --no-cpu > gpurun_out/${TAG}_k1c3_ncu.log 2>&1
echo "ncu rc=$?"
python profiles/summarize.py full /tmp/${TAG}_k1c3.ncu-rep > gpurun_out/${TAG}_k1c3_summary.md 2>&1
ncu -i /tmp/${TAG}_k1c3.ncu-rep --page source --csv --print-source sass > /tmp/${TAG}_k1c3_sass.csv 2>&1
python tools/sass_profile.py /tmp/${TAG}_k1c3_sass.csv > gpurun_out/${TAG}_k1c3_sass_profile.txt 2>&1
cp /tmp/${TAG}_k1c3.ncu-rep gpurun_out/ 2>/dev/null
cat gpurun_out/${TAG}_k1c3_summary.md | head -40
