#!/bin/bash
mkdir -p gpurun_out
T=${1:-k0ab2}
for L in build_trace/libmsort_k0_*.so; do
  echo "== $L"; MSORT_LIB=$L python scripts/graph_latency.py --sizes 13,14,15,16
done > gpurun_out/${T}.log 2>&1
echo "== trace 512x8x16" >> gpurun_out/${T}.log
MSORT_LIB=build_trace/libmsort_k0trace.so python scripts/k0_trace.py --log2n 16 >> gpurun_out/${T}.log 2>&1
cat gpurun_out/${T}.log
