mkdir -p gpurun_out
T=r2f
timeout 900 python -m pytest tests/test_gpu_sort.py tests/test_gpu_dist.py -x -q -k "small_cluster or c1 or emulated or nccl" > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${T}_pytest.log
tail -n 2 gpurun_out/${T}_pytest.log
timeout 300 python scripts/graph_latency.py --sizes 13,14,15,16 > gpurun_out/${T}_graph.log 2>&1; cat gpurun_out/${T}_graph.log
timeout 900 python bench.py --no-e2e --no-cpu-baseline --no-batched > gpurun_out/${T}_bench.log 2>&1; echo "bench rc=$?"
grep '^{' gpurun_out/${T}_bench.log | python3 -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['verified'])
c=d['configs']; print(c.get('t_C2s_over_C2'), c.get('t_C2r_over_C2'))
for k,v in c['results'].items(): print(k, v['ms'], v.get('graph_replay_ms'), v['verified'])"
