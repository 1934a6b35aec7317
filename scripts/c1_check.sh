mkdir -p gpurun_out
T=${1:-c1}
timeout 300 python scripts/graph_latency.py --sizes 12,14,16,17,18 > gpurun_out/${T}_graph.log 2>&1
cat gpurun_out/${T}_graph.log
python scripts/graph_latency.py --sizes 16 --reps 3 > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches.csv python scripts/graph_latency.py --sizes 16 --reps 3 > /dev/null 2>&1; echo "ncu rc=$?"
