# ncu launch list of the default bench command's timed region (128 steps opening on a refresh boundary)
set -x
TAG=${TAG:-r02}
ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${TAG}_launches_bench_default.csv python bench.py --no-cpu > gpurun_out/${TAG}_launches_bench.log 2>&1
echo "ncu rc=$?"
python profiles/summarize.py launches gpurun_out/${TAG}_launches_bench_default.csv
