# ncu --set full of the pairs tile sorts (C3: int64 + idx, C4: uint32 + idx) and their merge passes
mkdir -p gpurun_out; T=${1:-pairs}
for c in C3 C4; do
  python scripts/cfg_once.py $c --reps 2 > gpurun_out/${T}_${c}_plain.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"k1_tile_sort|k3_merge_pass" -s 2 -c 2 \
      -o gpurun_out/${T}_${c} python scripts/cfg_once.py $c --reps 2 > gpurun_out/${T}_${c}_ncu.log 2>&1
  echo "$c rc=$?"
done
