#!/bin/bash
mkdir -p gpurun_out
T=${1:-c2ab2}
for L in default build_trace/libmsort_pl1.so build_trace/libmsort_pl4.so; do
  if [ $L = default ]; then python scripts/c2_time.py --log2n 20 22 24 26; else MSORT_LIB=$L python scripts/c2_time.py --log2n 20 22 24 26; fi
done > gpurun_out/${T}.log 2>&1
MSORT_LIB=build_trace/libmsort_trace.so python scripts/k3_levels.py --log2n 24 --order random >> gpurun_out/${T}.log 2>&1
cat gpurun_out/${T}.log
