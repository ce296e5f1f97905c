# ncu --set full of the boundary's K-means kernels (first boundary of the timed window),
# plus raw metrics and SASS-level source page per kernel.
set -x
TAG=${TAG:-r02}
ncu --nvtx --nvtx-include "timed/" -k regex:"km_(prep|restart|table)" -c 24 --set full --clock-control none --import-source on \
    -o /tmp/${TAG}_km python bench.py --steps 8 --warmup 3 --no-cpu > gpurun_out/${TAG}_km_ncu.log 2>&1
echo "ncu rc=$?"
ncu -i /tmp/${TAG}_km.ncu-rep --page raw --csv > gpurun_out/${TAG}_km_raw.csv 2>&1
ncu -i /tmp/${TAG}_km.ncu-rep --page source --csv --print-source sass > gpurun_out/${TAG}_km_sass.csv 2>&1
TKV_KSTATS=1 python bench.py --steps 8 --warmup 3 --no-cpu > /dev/null 2> gpurun_out/${TAG}_kstats.txt
grep kstats gpurun_out/${TAG}_kstats.txt | tail -8
echo done
