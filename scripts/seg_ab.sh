#!/bin/bash
# batched + C1 A/B between library builds (bench lines)
mkdir -p gpurun_out
T=$1; shift
for L in "$@"; do
  if [ $L = default ]; then python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${T}_b.log 2>&1
  else MSORT_LIB=$L python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${T}_b.log 2>&1; fi
  L=$L T=$T python - <<'PY'
import json, os
L = [l for l in open("gpurun_out/%s_b.log" % os.environ["T"]).read().splitlines() if l.startswith("{")]
d = json.loads(L[-1])
c = d["configs"]["results"]["C1"]
print("==", os.environ["L"], "C1", c["ms"], c.get("graph_replay_ms"), "batched",
      {k: v["ms"] for k, v in d["batched_sort"]["results"].items()},
      all(v["verified"] for v in d["batched_sort"]["results"].values()), c["verified"])
PY
done 2>&1 | tee gpurun_out/${T}.log
python scripts/graph_latency.py --sizes 13,16 2>&1 | tee -a gpurun_out/${T}.log
MSORT_LIB=$2 python scripts/graph_latency.py --sizes 13,16 2>&1 | tee -a gpurun_out/${T}.log
