# end-of-round evidence on the final code: GPU suite + smoke + bench lines (final_validation.sh),
# config 1 line, then the K1 ncu capture (config 2 bench position) and the default window's launch list
set -x
TAG=${TAG:-r02}
bash tools/jobs/final_validation.sh
timeout 900 python bench.py --no-cpu --config 1 > gpurun_out/${TAG}_bench_c1.json 2> gpurun_out/${TAG}_bench_c1.err; echo "c1 rc=$?"
bash tools/jobs/k1_ncu.sh > /dev/null 2>&1; echo "k1 ncu rc=$?"
bash tools/jobs/launch_list.sh > gpurun_out/${TAG}_launches_summary.md 2>&1; echo "launch list rc=$?"
