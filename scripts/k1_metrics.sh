M=l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum,gpu__time_duration.sum,l1tex__throughput.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active
for lib in v_old libmsort; do
  MSORT_LIB=paper_2211_16479_b200/lib/$lib.so timeout 600 ncu --metrics $M --clock-control none -k regex:k1_tile -s 2 -c 1 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/k1m_$lib.txt 2>&1
done
