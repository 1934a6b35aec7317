# K0 multiway (MW) check: parity of every K0 size / dtype, graph latency MW vs level variant.
mkdir -p gpurun_out
T=${1:-k0mw}
timeout 600 python -m pytest tests/test_gpu_sort.py -x -q -k "small_cluster" > gpurun_out/${T}_sort.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_sort.log
tail -n 3 gpurun_out/${T}_sort.log
for m in 1 3; do echo "== MSORT_K0=$m"; MSORT_K0=$m timeout 300 python scripts/graph_latency.py --sizes 13,14,15,16 2>&1; done > gpurun_out/${T}_graph.log; cat gpurun_out/${T}_graph.log
