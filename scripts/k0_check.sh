mkdir -p gpurun_out
T=${1:-k0}
timeout 900 python -m pytest tests/test_gpu_sort.py -x -q > gpurun_out/${T}_sort.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_sort.log
MSORT_K0=2 timeout 900 python -m pytest tests/test_gpu_sort.py -x -q -k small_cluster > gpurun_out/${T}_sort2.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_sort2.log
tail -n 2 gpurun_out/${T}_sort.log gpurun_out/${T}_sort2.log
for m in 1 2 0; do echo "== MSORT_K0=$m"; MSORT_K0=$m timeout 300 python scripts/graph_latency.py --sizes 10,13,14,15,16 2>&1; done > gpurun_out/${T}_graph.log; cat gpurun_out/${T}_graph.log
