#!/bin/bash
# On the GPU box: GPU tests on the default build, then A/B of the variant libraries.
# Usage: bash scripts/ab_gpu.sh TAG lib1.so lib2.so ...
TAG=$1; shift
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
tail -n 2 gpurun_out/${TAG}_pytest.log
bash scripts/ab.sh paper_2211_16479_b200/lib/libmsort.so "$@" 2>&1 | tee gpurun_out/${TAG}_ab.log
