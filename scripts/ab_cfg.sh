#!/bin/bash
# configs_bench for each library variant: bash scripts/ab_cfg.sh lib...
for lib in "$@"; do echo "== $lib"; MSORT_LIB=$lib timeout 600 python scripts/configs_bench.py --reps 5 2>&1 | python3 -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print(d['config'], d['ms'], d['gkeys_s'], d['phase_ms'])"; done
