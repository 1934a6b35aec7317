#!/bin/bash
# configs A/B: per-config lines of bench.py for each library build given
mkdir -p gpurun_out
T=$1; shift
for L in "$@"; do
  if [ $L = default ]; then python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-batched > gpurun_out/${T}_b.log 2>&1
  else MSORT_LIB=$L python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-batched > gpurun_out/${T}_b.log 2>&1; fi
  L=$L T=$T python - <<'PY'
import json, os
d = json.loads(open("gpurun_out/%s_b.log" % os.environ["T"]).read().strip().splitlines()[-1])
print("==", os.environ["L"], "C5 ms", round(d["ms_per_step"], 4), "verified", d["verified"])
for k, v in d["configs"]["results"].items():
    print("  ", k, v["ms"], v.get("graph_replay_ms"), v["phases_ms"], v["verified"])
PY
done 2>&1 | tee gpurun_out/${T}.log
