"""L2 / memory-path metrics of an ncu report: ncu_l2.py rep"""
import csv, subprocess, sys
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr, units = rows[0], rows[1]
keys = ("lts__t_bytes.sum", "lts__t_sectors.sum", "lts__throughput.avg.pct", "lts__t_sectors_srcunit_tex",
        "lts__d_sectors", "l1tex__m_xbar2l1tex_read_bytes.sum", "l1tex__m_l1tex2xbar", "dram__bytes",
        "gpu__time_duration.sum", "sm__pipe_tensor_cycles_active.avg.pct", "lts__t_sector_hit_rate.pct",
        "gpu__compute_memory_throughput", "l1tex__throughput.avg.pct", "smsp__inst_executed.sum",
        "sm__cycles_elapsed.avg", "lts__cycles_elapsed.avg", "gpc__cycles_elapsed.max", "lts__t_requests",
        "smsp__average_warps_issue_stalled", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "smsp__cycles_active.avg", "sm__memory_throughput")
for r in rows[2:]:
    print("==", r[hdr.index("Kernel Name")][:90])
    for h, u, v in zip(hdr, units, r):
        if any(h.startswith(k) for k in keys) and not h.endswith(".per_second") and ".max." not in h and ".min." not in h:
            print(f"  {h:80s} {u:10s} {v}")
