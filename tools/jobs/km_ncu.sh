# ncu --set full of the boundary's K-means kernels (first boundary of the timed window);
# summaries are produced on the box (the SASS page of 24 K-means launches is ~200 MB).
set -x
TAG=${TAG:-r02}
ncu --nvtx --nvtx-include "timed/" -k regex:"km_(prep|restart|table)" -c 24 --set full --clock-control none --import-source on \
    -o /tmp/${TAG}_km python bench.py --steps 8 --warmup 3 --no-cpu > gpurun_out/${TAG}_km_ncu.log 2>&1
echo "ncu rc=$?"
python profiles/summarize.py full /tmp/${TAG}_km.ncu-rep > gpurun_out/${TAG}_km_summary.md 2>&1
ncu -i /tmp/${TAG}_km.ncu-rep --page source --csv --print-source sass > /tmp/${TAG}_km_sass.csv 2>&1
python tools/sass_profile.py /tmp/${TAG}_km_sass.csv > gpurun_out/${TAG}_km_sass_profile.txt 2>&1
TKV_KSTATS=1 python bench.py --steps 8 --warmup 3 --no-cpu > /dev/null 2> gpurun_out/${TAG}_kstats.txt
grep kstats gpurun_out/${TAG}_kstats.txt | tail -8
echo done
