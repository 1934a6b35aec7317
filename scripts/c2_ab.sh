#!/bin/bash
# C2 A/B: trace + per-config timings of the current build.
mkdir -p gpurun_out
T=${1:-c2ab}
MSORT_LIB=build_trace/libmsort_trace.so python scripts/k3_levels.py --log2n 24 --order random > gpurun_out/${T}_trace.log 2>&1
MSORT_LIB=build_trace/libmsort_trace.so python scripts/k3_levels.py --log2n 24 --order sorted >> gpurun_out/${T}_trace.log 2>&1
python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-batched > gpurun_out/${T}_bench.log 2>&1
T=$T python - <<'PY' >> gpurun_out/${T}_trace.log
import json, os
d = json.loads(open("gpurun_out/%s_bench.log" % os.environ["T"]).read().strip().splitlines()[-1])
print("C5 ms", round(d["ms_per_step"], 4), "verified", d["verified"])
for k, v in d["configs"]["results"].items():
    print(k, v["ms"], v.get("graph_replay_ms"), v["phases_ms"], v["verified"])
PY
cat gpurun_out/${T}_trace.log
