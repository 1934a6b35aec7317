#!/bin/bash
# Tuning round: quick size sweep, bench per-config lines, GPU tests.
mkdir -p gpurun_out
T=${1:-ab}
python scripts/c2_time.py --log2n 20 22 24 26 27 28 --reps 10 > gpurun_out/${T}_sizes.log 2>&1
python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${T}_bench.log 2>&1
T=$T python - <<'PY' >> gpurun_out/${T}_sizes.log
import json, os
d = json.loads(open("gpurun_out/%s_bench.log" % os.environ["T"]).read().strip().splitlines()[-1])
print("C5 ms", round(d["ms_per_step"], 4), "verified", d["verified"])
for k, v in d["configs"]["results"].items():
    print(k, v["ms"], v.get("graph_replay_ms"), v["phases_ms"], v["verified"])
print("batched", d["batched_sort"]["results"])
PY
cat gpurun_out/${T}_sizes.log
if [ "$2" = tests ]; then timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -3; fi
