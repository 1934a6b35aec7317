"""Print ms/step, verified and phases of a bench.py JSON log (last line).

    python scripts/bench_summary.py LOG [LABEL]
"""
import json
import sys

d = json.loads([x for x in open(sys.argv[1]) if x.startswith("{")][-1])
print(sys.argv[2] if len(sys.argv) > 2 else "", round(d["ms_per_step"], 4), d["verified"],
      {k: v["ms_per_step"] for k, v in d["phases"].items()}, d["clocks"].get("sm_mhz"))
