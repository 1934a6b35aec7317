mkdir -p gpurun_out
T=${1:-k5ab}
timeout 900 python -m pytest tests/test_gpu_merge.py -x -q > gpurun_out/${T}_merge.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_merge.log
tail -n 2 gpurun_out/${T}_merge.log
for v in "" _k5g4 _k5g12; do
  echo "== lib$v" >> gpurun_out/${T}.log
  MSORT_LIB=$PWD/paper_2211_16479_b200/lib/libmsort$v.so timeout 300 python scripts/k5_bench.py --ps 3,4,8,16 >> gpurun_out/${T}.log 2>&1
done
cat gpurun_out/${T}.log
