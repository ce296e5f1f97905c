#!/bin/bash
timeout 600 python scratch/kstats_run.py 1536 4 nostats 2>&1 | tail -2
TKV_KM64_256=1 timeout 600 python scratch/kstats_run.py 1536 4 nostats 2>&1 | tail -2
TKV_KM64_256=1 timeout 600 python -m pytest tests -m gpu -x -q -k "kmeans or llama or calibrated" 2>&1 | tail -2
timeout 900 python -m pytest tests -m gpu -x -q > /dev/null 2>&1; echo "full gpu suite rc=$?"
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "sparsity_trace" 2>&1 | tail -3
