#!/bin/bash
# A/B the library variants on the bench workload: prints merge_pass avg ms and ms/step.
for lib in "$@"; do
  out=$(MSORT_LIB=$lib timeout 300 python bench.py --no-e2e --no-cpu-baseline --steps 10 --warmup 3 2>/dev/null | tail -1)
  python3 - "$lib" "$out" <<'PY'
import json,sys
lib,out=sys.argv[1],sys.argv[2]
try:
    d=json.loads(out)
    ph=d["phases"]
    print(f"{lib.split('/')[-1]:28s} ms/step={d['ms_per_step']:.3f} Gk/s={d['value']/1e9:.2f} merge_total={ph['merge_pass']['ms_per_step']:.4f} per_level={ph['merge_pass']['ms_per_step']/d['config']['merge_passes']:.4f} tile={ph['tile_sort']['ms_per_step']:.3f} frac={d['roofline']['frac']} ok={d['verified']}")
except Exception as e:
    print(lib, "FAILED", out[:300])
PY
done
