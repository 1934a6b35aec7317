#!/bin/bash
# Evidence run after K0 multiway: GPU tests, smoke, bench, ncu launch list, ncu --set full of K0 (C1).
T=${1:-r2k}
bash scripts/gpu_check.sh $T
python scripts/one_sort.py --log2n 16 --seed 0 --reps 4 > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k0_small_sort -s 3 -c 1 -o gpurun_out/${T}_k0 \
  python scripts/one_sort.py --log2n 16 --seed 0 --reps 4 > gpurun_out/${T}_ncu_k0.log 2>&1
echo "ncu k0 rc=$?"
timeout 300 python scripts/graph_latency.py --sizes 10,13,14,15,16 > gpurun_out/${T}_graph.log 2>&1; cat gpurun_out/${T}_graph.log
