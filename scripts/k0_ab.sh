#!/bin/bash
mkdir -p gpurun_out
T=${1:-k0ab}
for L in default build_trace/libmsort_k0_*.so; do
  echo "== $L"
  if [ $L = default ]; then python scripts/graph_latency.py --sizes 10,13,14,15,16; else MSORT_LIB=$L python scripts/graph_latency.py --sizes 10,13,14,15,16; fi
done > gpurun_out/${T}.log 2>&1
cat gpurun_out/${T}.log
