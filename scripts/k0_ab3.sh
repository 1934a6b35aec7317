# K0 MW A/B: trace (fixed marks), VT2 = 12 vs 16, level variant
mkdir -p gpurun_out; T=${1:-k0ab3}; L=$PWD/paper_2211_16479_b200/lib
MSORT_LIB=$L/libmsort_k0trace.so python scripts/k0_trace.py --log2n 16 > gpurun_out/${T}_trace.log 2>&1
for v in libmsort.so libmsort_k0vt16.so; do echo "== $v"; MSORT_LIB=$L/$v timeout 300 python scripts/graph_latency.py --sizes 13,14,15,16 2>&1; done > gpurun_out/${T}_graph.log
echo "== level variant"; MSORT_K0=3 python scripts/graph_latency.py --sizes 16 >> gpurun_out/${T}_graph.log 2>&1
cat gpurun_out/${T}_graph.log; head -2 gpurun_out/${T}_trace.log
