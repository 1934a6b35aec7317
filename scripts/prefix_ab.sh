# K3 top-level prefix dependency: parity, level trace, C5 A/B against the previous build
mkdir -p gpurun_out; T=${1:-pfx}; L=$PWD/paper_2211_16479_b200/lib
timeout 900 python -m pytest tests/test_gpu_sort.py tests/test_gpu_workspace.py tests/test_gpu_graph.py -x -q > gpurun_out/${T}_tests.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_tests.log; tail -n 2 gpurun_out/${T}_tests.log
MSORT_LIB=$L/libmsort_k3trace.so timeout 300 python scripts/k3_levels.py --log2n 28 --seed 4 > gpurun_out/${T}_lv28.log 2>&1; tail -n 4 gpurun_out/${T}_lv28.log
B="python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --no-batched --no-configs"
for r in 1 2; do for v in libmsort_prev.so libmsort.so; do echo "== $v"; MSORT_LIB=$L/$v timeout 300 $B 2>&1 | python -c "import sys,json; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); print(round(d['ms_per_step'],4), d['roofline']['avg_launch_ms'], d['verified'], d['clocks']['reasons'])"; done; done > gpurun_out/${T}_ab.log 2>&1; cat gpurun_out/${T}_ab.log
