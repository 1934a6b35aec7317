mkdir -p gpurun_out
T=${1:-k1ab}
python scripts/k1_ab.py > gpurun_out/${T}.log 2>&1; cat gpurun_out/${T}.log
python scripts/k1_ab.py --reps 1 > /dev/null 2>&1 && ncu --set full --clock-control none -k regex:k1_tile_sort_keys -s 3 -c 2 -o gpurun_out/${T}_prof python scripts/k1_ab.py --reps 1 > gpurun_out/${T}_ncu.log 2>&1; echo "ncu rc=$?"
