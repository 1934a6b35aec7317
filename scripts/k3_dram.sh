#!/bin/bash
# DRAM bytes and duration of one fused K3 launch per library variant (bench workload).
# Usage: bash scripts/k3_dram.sh TAG lib1.so lib2.so ...
TAG=$1; shift
mkdir -p gpurun_out
for lib in "$@"; do
  MSORT_LIB=$lib timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
    --clock-control none -k regex:k3_merge -s 1 -c 1 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline \
    > gpurun_out/${TAG}_$(basename $lib .so).txt 2>&1
  echo "$(basename $lib): $(grep -E 'dram__bytes|duration' gpurun_out/${TAG}_$(basename $lib .so).txt | awk '{print $1, $(NF)}' | tr '\n' ' ')"
done
