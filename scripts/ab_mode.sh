#!/bin/bash
# A/B library variants with an environment mode: bash scripts/ab_mode.sh "ENV=..." lib...
ENVS=$1; shift
for lib in "$@"; do
  out=$(env $ENVS MSORT_LIB=$lib timeout 300 python bench.py --no-e2e --no-cpu-baseline --steps 10 --warmup 3 2>/dev/null | grep "^{")
  python3 - "$lib" "$out" <<'PY'
import json,sys
lib,out=sys.argv[1],sys.argv[2]
try:
    d=json.loads(out); ph=d["phases"]
    print(f"{lib.split('/')[-1]:32s} ms/step={d['ms_per_step']:.3f} merge={ph['merge_pass']['ms_per_step']:.3f} tile={ph['tile_sort']['ms_per_step']:.3f} ok={d['verified']}")
except Exception as e:
    print(lib, "FAILED", out[:200])
PY
done
