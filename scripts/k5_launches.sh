mkdir -p gpurun_out
T=${1:-k5l}
python scripts/k5_bench.py --ps 8,16 --reps 1 > gpurun_out/${T}_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k5_ --csv --log-file gpurun_out/${T}_launches.csv python scripts/k5_bench.py --ps 8,16 --reps 1 > gpurun_out/${T}_ncu.log 2>&1
echo "ncu rc=$?"
