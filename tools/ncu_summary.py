"""Summarise ncu reports: python tools/ncu_summary.py rep1.ncu-rep [...]"""
import csv, subprocess, sys, io
KEYS = [
 ("gpu__time_duration.sum", "duration"),
 ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM %"),
 ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
 ("smsp__thread_inst_executed_per_inst_executed.ratio", "active threads/warp"),
 ("sm__warps_active.avg.per_cycle_active", "warps active/SM"),
 ("launch__registers_per_thread", "regs"),
 ("launch__grid_size", "grid"),
 ("l1tex__t_sector_hit_rate.pct", "L1 hit %"),
 ("lts__t_sector_hit_rate.pct", "L2 hit %"),
 ("dram__bytes_read.sum", "DRAM read"),
 ("dram__bytes_write.sum", "DRAM write"),
 ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe %"),
 ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU pipe %"),
 ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe %"),
 ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe %"),
 ("smsp__inst_executed.sum", "warp inst"),
 ("smsp__thread_inst_executed.sum", "thread inst"),
 ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem wavefronts"),
 ("lts__t_sectors.sum", "L2 sectors"),
 ("l1tex__t_sectors.sum", "L1 sectors"),
]
STALL = "smsp__average_warps_issue_stalled_"
for rep in sys.argv[1:]:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    print("==", rep)
    for v in rows[2:]:
        print("  kernel:", v[h.index("Kernel Name")][:90])
        for k, name in KEYS:
            if k in h:
                i = h.index(k)
                print(f"    {name:22s} {v[i]} {units[i]}")
        st = [(h[i][len(STALL):].replace("_per_issue_active.ratio", ""), float(v[i])) for i in range(len(h))
              if h[i].startswith(STALL) and h[i].endswith("per_issue_active.ratio") and v[i]]
        st.sort(key=lambda x: -x[1])
        print("    stalls/issue:", ", ".join(f"{n}={x:.2f}" for n, x in st[:8]))
