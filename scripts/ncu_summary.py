"""Summarise an ncu --page raw --csv export: key counters per kernel.

    ncu -i X.ncu-rep --page raw --csv > X_raw.csv; python scripts/ncu_summary.py X_raw.csv
"""
import csv
import sys

WANT = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'lts__t_bytes.sum', 'dram__throughput.avg.pct_of_peak_sustained_elapsed',
        'sm__throughput.avg.pct_of_peak_sustained_elapsed',
        'l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum',
        'l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum',
        'l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum',
        'l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum',
        'smsp__inst_executed.sum', 'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'sm__warps_active.avg.pct_of_peak_sustained_active',
        'l1tex__throughput.avg.pct_of_peak_sustained_active', 'launch__registers_per_thread',
        'launch__grid_size', 'launch__block_size']
rows = list(csv.reader(open(sys.argv[1])))
hdr, units, data = rows[0], rows[1], rows[2:]
for d in data:
    print('-----', d[hdr.index('Kernel Name')][:110])
    for w in WANT:
        if w in hdr:
            i = hdr.index(w)
            print(f"  {w:62s} {d[i]:>18s} {units[i]}")
    st = [(h, d[i]) for i, h in enumerate(hdr) if h.startswith('smsp__pcsamp_warps_issue_stalled_')
          and not h.endswith('_not_issued')]
    tot = sum(float(v.replace(',', '')) for _, v in st if v)
    top = sorted(st, key=lambda x: -float(x[1].replace(',', '') or 0))[:8]
    print('  stalls (pc sampling):', ', '.join(f"{h[33:]} {100*float(v.replace(',',''))/tot:.0f}%"
                                              for h, v in top if tot))
