# One ncu --set full capture of K1 at the bench position (between boundaries),
# with source correlation, plus a SASS-level source page for instruction counts.
set -x
TAG=${TAG:-r02}
ncu --nvtx --nvtx-include "timed/" -k regex:"attend_" -s 2 -c 1 --set full --clock-control none --import-source on \
    -o /tmp/${TAG}_k1 python bench.py --steps 8 --warmup 3 --no-cpu > gpurun_out/${TAG}_k1_ncu.log 2>&1
echo "ncu rc=$?"
ncu -i /tmp/${TAG}_k1.ncu-rep --page raw --csv > gpurun_out/${TAG}_k1_raw.csv 2>&1
ncu -i /tmp/${TAG}_k1.ncu-rep --page source --csv --print-source sass > gpurun_out/${TAG}_k1_sass.csv 2>&1
echo done
