#!/bin/bash
# quick.sh, then (if it passed) ncu --set full of one launch of the kernels matching $2.
# Usage: bash scripts/quick_prof.sh TAG REGEX
TAG=$1; RX=$2
bash scripts/quick.sh $TAG
if grep -q "pytest rc=0" gpurun_out/${TAG}_pytest.log; then
  CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
  $CMD > gpurun_out/${TAG}_plain.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$RX" -s 3 -c 1 \
    -o gpurun_out/${TAG} $CMD > gpurun_out/${TAG}_ncu.log 2>&1
  echo "ncu rc=$?"
fi
