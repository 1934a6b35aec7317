#!/bin/bash
# latency per size for each library variant: bash scripts/ab_lat.sh SIZES lib...
SZ=$1; shift
for lib in "$@"; do echo "== $lib"; MSORT_LIB=$lib timeout 300 python scripts/latency.py --sizes $SZ --reps 20 2>&1 | python3 -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print(d['log2n'], d['ms'], d['gkeys_s'], d['phase_ms'])"; done
