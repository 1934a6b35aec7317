#!/bin/bash
mkdir -p gpurun_out
T=${1:-c2ab4}
for L in default build_trace/libmsort_g1c2.so build_trace/libmsort_g1c3.so build_trace/libmsort_g1c4.so; do
  if [ $L = default ]; then python scripts/c2_time.py --log2n 24 26 27 28 --reps 10; else MSORT_LIB=$L python scripts/c2_time.py --log2n 24 26 27 28 --reps 10; fi
done > gpurun_out/${T}.log 2>&1
cat gpurun_out/${T}.log
