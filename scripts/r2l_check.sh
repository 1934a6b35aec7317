#!/bin/bash
# Session-4 evidence run: GPU tests, smoke, bench, ncu launch list; ncu --set full of
# K1/K3 (C5), K5 (p = 8), K0 (C1) and the C3 narrowed path (range / narrow / widen + 4-byte K1/K3).
# Reports are exported to raw CSV on the box and deleted (gpurun copies back <= 64 MiB).
T=${1:-r2l}
PART=${2:-all}
raw() { ncu -i gpurun_out/$1.ncu-rep --page raw --csv > gpurun_out/$1_raw.csv 2>/dev/null; rm -f gpurun_out/$1.ncu-rep; }
if [ "$PART" = all ] || [ "$PART" = a ] || [ "$PART" = c ]; then
bash scripts/gpu_check.sh $T
fi
if [ "$PART" = all ] || [ "$PART" = a ]; then
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-batched --no-configs"
$B > /dev/null 2>&1 && ncu --set full --clock-control none -k regex:"k1_tile_sort_keys|k3_merge_pass" -s 6 -c 2 -o gpurun_out/${T}_k1k3 $B > gpurun_out/${T}_ncu_full.log 2>&1
echo "ncu k1k3 rc=$?"; raw ${T}_k1k3
ncu --set full --clock-control none -k regex:k0_small_sort -s 3 -c 1 -o gpurun_out/${T}_k0 \
  python scripts/one_sort.py --log2n 16 --seed 0 --reps 4 > gpurun_out/${T}_ncu_k0.log 2>&1
echo "ncu k0 rc=$?"; raw ${T}_k0
timeout 300 python scripts/graph_latency.py --sizes 10,13,14,15,16 > gpurun_out/${T}_graph.log 2>&1; cat gpurun_out/${T}_graph.log
fi
if [ "$PART" = all ] || [ "$PART" = b ]; then
python scripts/k5_bench.py --ps 8 --reps 1 > /dev/null 2>&1 && ncu --set full --clock-control none -k regex:k5_merge -s 3 -c 1 -o gpurun_out/${T}_k5 python scripts/k5_bench.py --ps 8 --reps 1 > gpurun_out/${T}_ncu_k5.log 2>&1
echo "ncu k5 rc=$?"; raw ${T}_k5
fi
if [ "$PART" = all ] || [ "$PART" = b ] || [ "$PART" = c ]; then
ncu --set full --clock-control none -k regex:"k_key_|k1_tile_sort|k3_merge_pass" -s 7 -c 7 -o gpurun_out/${T}_c3 \
  python scripts/cfg_once.py C3 --reps 2 > gpurun_out/${T}_ncu_c3.log 2>&1
echo "ncu c3 rc=$?"; raw ${T}_c3
fi
du -sh gpurun_out
