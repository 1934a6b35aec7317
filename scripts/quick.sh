#!/bin/bash
# Quick GPU iteration: GPU parity tests then a short bench.  Usage: bash scripts/quick.sh TAG [pytest -k expr]
TAG=${1:-q}; K=${2:-}
mkdir -p gpurun_out
if [ -n "$K" ]; then timeout 900 python -m pytest tests -m gpu -x -q -k "$K" > gpurun_out/${TAG}_pytest.log 2>&1
else timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest.log 2>&1; fi
echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
tail -n 3 gpurun_out/${TAG}_pytest.log
timeout 300 python bench.py --no-e2e --no-cpu-baseline --steps 20 --warmup 5 > gpurun_out/${TAG}_bench.log 2>&1
python3 - gpurun_out/${TAG}_bench.log <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    ph=d["phases"]
    print(f"ms/step={d['ms_per_step']:.3f} Gk/s={d['value']/1e9:.2f} " + " ".join(f"{k}={v['ms_per_step']:.3f}" for k,v in ph.items()) + f" frac={d['roofline']['frac']} ok={d['verified']} clk={d['clocks'].get('sm_mhz')}")
except Exception as e:
    print("bench FAILED", open(sys.argv[1]).read()[-2000:])
PY
