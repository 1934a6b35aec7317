#!/bin/bash
# Round-2 evidence run: GPU tests, smoke, bench, ncu launch list, ncu --set full of K1/K3/K5.
T=${1:-r2full}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${T}_smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${T}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${T}_smoke.log
timeout 900 python bench.py > gpurun_out/${T}_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/${T}_bench.log
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-batched --no-configs"
$B > gpurun_out/${T}_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${T}_launches.csv $B > gpurun_out/${T}_ncu_list.log 2>&1
echo "ncu list rc=$?"
$B > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"k1_tile_sort_keys|k3_merge_pass" -s 6 -c 2 -o gpurun_out/${T}_k1k3 $B > gpurun_out/${T}_ncu_full.log 2>&1
echo "ncu full rc=$?"
python scripts/k5_bench.py --ps 8 --reps 1 > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k5_merge -s 3 -c 1 -o gpurun_out/${T}_k5 python scripts/k5_bench.py --ps 8 --reps 1 > gpurun_out/${T}_ncu_k5.log 2>&1
echo "ncu k5 rc=$?"
tail -n 2 gpurun_out/${T}_pytest.log gpurun_out/${T}_smoke.log; tail -c 400 gpurun_out/${T}_bench.log
