#!/bin/bash
for L in default build_trace/libmsort_ring3.so build_trace/libmsort_ring4.so default; do
  if [ $L = default ]; then python scripts/c2_time.py --log2n 20 22 24 26 27 --reps 15; else MSORT_LIB=$L python scripts/c2_time.py --log2n 20 22 24 26 27 --reps 15; fi
done 2>&1 | grep random | tee gpurun_out/ring_ab.log
