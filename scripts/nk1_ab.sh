# narrowing folded into K1: parity + C3 A/B
mkdir -p gpurun_out; T=${1:-nk1}; L=$PWD/paper_2211_16479_b200/lib
timeout 900 python -m pytest tests/test_gpu_sort.py tests/test_gpu_graph.py tests/test_gpu_workspace.py tests/test_gpu_dist.py -x -q > gpurun_out/${T}_tests.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_tests.log; tail -n 2 gpurun_out/${T}_tests.log
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-batched"
for v in libmsort_prev.so libmsort.so libmsort_prev.so libmsort.so; do echo "== $v"; MSORT_LIB=$L/$v timeout 600 $B 2>&1 | python -c "
import sys,json
d=json.loads([l for l in sys.stdin if l.startswith('{')][-1])
r=d['configs']['results']
print({k: (r[k]['ms'], r[k]['phases_ms'], r[k]['verified']) for k in ('C3',)})"; done > gpurun_out/${T}_ab.log 2>&1; cat gpurun_out/${T}_ab.log
