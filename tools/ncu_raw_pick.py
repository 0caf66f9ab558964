"""Print selected metrics of an `ncu --page raw --csv` export, one column per launch.
usage: python tools/ncu_raw_pick.py raw.csv [substring ...]"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
h, u = rows[0], rows[1]
pick = sys.argv[2:] or ["gpu__time_duration.sum", "smsp__inst_executed.sum", "smsp__issue_active.avg.pct", "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active",
                        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.per_cycle_active", "launch__registers_per_thread",
                        "issue_stalled", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct", "launch__occupancy_limit"]
ki = h.index("Kernel Name")
print("kernel".ljust(70), [r[ki][:40] for r in rows[2:]])
for i, name in enumerate(h):
    if any(p in name for p in pick) and "pcsamp" not in name and "not_issued" not in name:
        print(name[:68].ljust(70), u[i][:8].ljust(8), [r[i] for r in rows[2:] if len(r) > i])
