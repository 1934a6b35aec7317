mkdir -p gpurun_out
T=${1:-q}
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${T}_pytest.log
tail -n 3 gpurun_out/${T}_pytest.log
timeout 300 python scripts/dist_emul_bench.py --log2n 26 --ps 2,4,8 > gpurun_out/${T}_emul.log 2>&1; cat gpurun_out/${T}_emul.log
timeout 300 python scripts/k5_bench.py --ps 3,4,8 > gpurun_out/${T}_k5.log 2>&1; cat gpurun_out/${T}_k5.log
