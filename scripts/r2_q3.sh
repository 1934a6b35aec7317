mkdir -p gpurun_out
T=r2g
timeout 600 python -m pytest tests/test_gpu_dist.py -x -q -k "skewed" > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${T}_pytest.log
tail -n 2 gpurun_out/${T}_pytest.log
timeout 600 python bench.py --distributed-path --steps 5 --warmup 3 > gpurun_out/${T}_dbench.log 2>&1; echo "dbench rc=$?"
tail -c 1500 gpurun_out/${T}_dbench.log
