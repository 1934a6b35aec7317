mkdir -p gpurun_out; T=${1:-k0ab4}; L=$PWD/paper_2211_16479_b200/lib
timeout 600 python -m pytest tests/test_gpu_sort.py -x -q -k "small_cluster" > gpurun_out/${T}_sort.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_sort.log; tail -n 2 gpurun_out/${T}_sort.log
MSORT_LIB=$L/libmsort_k0trace.so python scripts/k0_trace.py --log2n 16 > gpurun_out/${T}_trace.log 2>&1
timeout 300 python scripts/graph_latency.py --sizes 13,14,15,16 > gpurun_out/${T}_graph.log 2>&1
cat gpurun_out/${T}_graph.log; head -2 gpurun_out/${T}_trace.log
