mkdir -p gpurun_out
T=${1:-k5n}
python scripts/k5_bench.py --ps 8 --reps 1 > gpurun_out/${T}_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k5_merge -s 3 -c 1 -o gpurun_out/${T}_prof python scripts/k5_bench.py --ps 8 --reps 1 > gpurun_out/${T}_ncu.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/${T}_ncu.log
