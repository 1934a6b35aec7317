#!/bin/bash
# ncu --set full of the batched-sort kernels (scripts/seg_prof.py).  Usage: bash scripts/ncu_seg.sh TAG
TAG=${1:-seg}
mkdir -p gpurun_out
python scripts/seg_prof.py > gpurun_out/${TAG}_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"kseg_warp_sort|k1_tile_sort|k3_merge_pass|kseg_classify" -c 8 \
  -o gpurun_out/${TAG} python scripts/seg_prof.py > gpurun_out/${TAG}_ncu.log 2>&1
echo "rc=$?"; tail -3 gpurun_out/${TAG}_ncu.log
