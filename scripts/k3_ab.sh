#!/bin/bash
mkdir -p gpurun_out
T=${1:-k3ab}
for L in default build_trace/libmsort_k3_*.so; do
  if [ $L = default ]; then python scripts/c2_time.py --log2n 24 26 28 --reps 10; else MSORT_LIB=$L python scripts/c2_time.py --log2n 24 26 28 --reps 10; fi
done > gpurun_out/${T}.log 2>&1
cat gpurun_out/${T}.log
