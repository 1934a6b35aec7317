#!/bin/bash
# t(C2s)/t(C2) diagnosis -- K1 and K3 counters on C2 random / sorted / reversed.
mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,lts__t_sector_hit_rate.pct,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum,sm__inst_executed.sum,smsp__inst_executed_op_shared_ld.sum,l1tex__throughput.avg.pct_of_peak_sustained_elapsed,sm__throughput.avg.pct_of_peak_sustained_elapsed,dram__throughput.avg.pct_of_peak_sustained_elapsed
for o in random sorted reversed; do
  python scripts/one_sort.py --log2n 24 --order $o --reps 4 > /dev/null 2>&1 && \
  ncu --metrics $M --clock-control none -k regex:"k1_tile_sort_keys|k3_merge_pass" -s 6 -c 2 --csv \
    python scripts/one_sort.py --log2n 24 --order $o --reps 4 > gpurun_out/c2_ncu_$o.csv 2> gpurun_out/c2_ncu_$o.err
  echo "$o rc=$?"
done
