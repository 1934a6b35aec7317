# top-level prefix waits (block counters): parity + C5 / configs A/B
mkdir -p gpurun_out; T=${1:-topblk}; L=$PWD/paper_2211_16479_b200/lib
timeout 900 python -m pytest tests/test_gpu_sort.py tests/test_gpu_graph.py tests/test_gpu_workspace.py tests/test_gpu_large.py -x -q > gpurun_out/${T}_tests.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_tests.log; tail -n 2 gpurun_out/${T}_tests.log
B="python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --no-batched"
for r in 1 2; do for v in libmsort_prev.so libmsort.so; do echo "== $v"; MSORT_LIB=$L/$v timeout 600 $B 2>&1 | python -c "
import sys,json
d=json.loads([l for l in sys.stdin if l.startswith('{')][-1])
r=d['configs']['results']
print(round(d['ms_per_step'],4), d['roofline']['avg_launch_ms'], d['verified'], d['clocks']['reasons'], {k: (r[k]['ms'], r[k]['verified']) for k in ('C1','C2','C2s','C2r','C3','C4')})"; done; done > gpurun_out/${T}_ab.log 2>&1; cat gpurun_out/${T}_ab.log
