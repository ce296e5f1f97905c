# ncu --set full captures of the final K1 and K-means kernels at the bench position
set -x
TAG=${TAG:-r02}
TAG=$TAG bash tools/jobs/k1_ncu.sh
TAG=$TAG bash tools/jobs/km_ncu.sh
ls -la gpurun_out/ | tail -20
