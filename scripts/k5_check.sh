mkdir -p gpurun_out
T=${1:-k5}
timeout 900 python -m pytest tests/test_gpu_merge.py -x -q > gpurun_out/${T}_merge.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_merge.log
timeout 300 python scripts/k5_bench.py --ps 3,4,8,16 > gpurun_out/${T}_bench.log 2>&1
timeout 900 python -m pytest tests/test_gpu_dist.py -x -q > gpurun_out/${T}_dist.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_dist.log
tail -n 2 gpurun_out/${T}_merge.log gpurun_out/${T}_dist.log; cat gpurun_out/${T}_bench.log
