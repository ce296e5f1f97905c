#!/bin/bash
timeout 600 python scratch/k1bench.py 2600 v3,minb4 2>&1 | tail -7
