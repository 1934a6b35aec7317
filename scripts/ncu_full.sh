#!/bin/bash
# ncu --set full of K1 and the fused K3 on the bench workload (one GPU).  Usage: bash scripts/ncu_full.sh TAG [bench args]
TAG=${1:-prof}; shift
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline $*"
$CMD > gpurun_out/${TAG}_plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k1_tile_sort|k3_merge_pass" -s 6 -c 2 \
  -o gpurun_out/${TAG} $CMD > gpurun_out/${TAG}_ncu.log 2>&1
echo "rc=$?"; tail -3 gpurun_out/${TAG}_ncu.log
