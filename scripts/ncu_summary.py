"""Print the key metrics of an ncu report (first kernel): usage ncu_summary.py rep [filter...]"""
import csv, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr, units = rows[0], rows[1]
want = sys.argv[2:] or ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active', 'smsp__inst_executed.sum',
        'sm__warps_active.avg.pct', 'launch__registers_per_thread', 'l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op',
        'l1tex__data_pipe_lsu_wavefronts_mem_shared_op', 'smsp__issue_active.avg.pct', 'smsp__average_warps_issue_stalled',
        'sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active', 'sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active',
        'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active', 'lts__t_bytes.sum', 'sm__throughput.avg.pct',
        'l1tex__t_bytes_pipe_lsu_mem_global_op_ld.sum', 'launch__grid_size', 'launch__waves']
for r in rows[2:]:
    print("==", r[hdr.index("Kernel Name")][:80])
    for h, u, v in zip(hdr, units, r):
        if any(h.startswith(w) for w in want):
            if 'stalled' in h:
                try:
                    if float(v) < 0.1: continue
                except ValueError:
                    pass
            if h.endswith('.per_second') or '.max.' in h or '.min.' in h or '.sum.pct' in h: continue
            print(f"  {h:75s} {u:10s} {v}")
