# Launch list of the timed window that opens on the tau boundary (ncu, cold/serialised)
# and the in-kernel K-means phase counters of the same window.
set -x
TAG=${TAG:-r02}
ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${TAG}_launches_boundary.csv python bench.py --steps 8 --warmup 3 --no-cpu --e2e-steps 128 > gpurun_out/${TAG}_ncu_bench.log 2>&1
echo "ncu rc=$?"
TKV_KSTATS=1 python bench.py --steps 8 --warmup 3 --no-cpu > gpurun_out/${TAG}_kstats.json 2> gpurun_out/${TAG}_kstats.txt
echo "kstats rc=$?"
grep kstats gpurun_out/${TAG}_kstats.txt | tail -20
