#!/bin/bash
# Per-level K3 timeline for C2 (2^24) random / sorted / reversed and C5 (2^28).
mkdir -p gpurun_out
export MSORT_LIB=build_trace/libmsort_trace.so
for o in random sorted reversed; do python scripts/k3_levels.py --log2n 24 --order $o; done > gpurun_out/c2_trace.log 2>&1
python scripts/k3_levels.py --log2n 28 --seed 4 >> gpurun_out/c2_trace.log 2>&1
cat gpurun_out/c2_trace.log
