# One ncu --set full capture of K1 at the bench position (first timed step = a refresh
# boundary), summarised on the box: key counters, stall reasons, SASS opcode histogram.
set -x
TAG=${TAG:-r02}
ncu --nvtx --nvtx-include "timed/" -k regex:"attend_" -c 1 --set full --clock-control none --import-source on \
    -o /tmp/${TAG}_k1 python bench.py --steps 8 --warmup 3 --no-cpu > gpurun_out/${TAG}_k1_ncu.log 2>&1
echo "ncu rc=$?"
python profiles/summarize.py full /tmp/${TAG}_k1.ncu-rep > gpurun_out/${TAG}_k1_summary.md 2>&1
ncu -i /tmp/${TAG}_k1.ncu-rep --page raw --csv > gpurun_out/${TAG}_k1_raw.csv 2>&1
ncu -i /tmp/${TAG}_k1.ncu-rep --page source --csv --print-source sass > /tmp/${TAG}_k1_sass.csv 2>&1
python tools/sass_profile.py /tmp/${TAG}_k1_sass.csv > gpurun_out/${TAG}_k1_sass_profile.txt 2>&1
cat gpurun_out/${TAG}_k1_summary.md
echo done
