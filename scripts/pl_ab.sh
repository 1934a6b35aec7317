#!/bin/bash
mkdir -p gpurun_out
for L in default build_trace/libmsort_pl2.so default build_trace/libmsort_pl2.so; do
  if [ $L = default ]; then python scripts/c2_time.py --log2n 22 24 26 --reps 20; else MSORT_LIB=$L python scripts/c2_time.py --log2n 22 24 26 --reps 20; fi
done 2>&1 | tee gpurun_out/pl_ab.log
