# K1 (keys, 2^28 int32) ncu --set full with source: per-line shared-memory wavefronts / conflicts
mkdir -p gpurun_out; T=${1:-k1src}
B="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-batched --no-configs"
$B > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k1_tile_sort_keys -s 3 -c 1 -o gpurun_out/${T} $B > gpurun_out/${T}_ncu.log 2>&1
echo "ncu rc=$?"
ncu -i gpurun_out/${T}.ncu-rep --page source --csv --print-source sass,cuda > gpurun_out/${T}_source.csv 2>/dev/null
ncu -i gpurun_out/${T}.ncu-rep --page source --csv > gpurun_out/${T}_source_cuda.csv 2>/dev/null
rm -f gpurun_out/${T}.ncu-rep
ls -la gpurun_out/${T}_*; du -sh gpurun_out
