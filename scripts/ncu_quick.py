"""Key counters of one kernel from `ncu -i REP --page raw --csv`."""
import csv, subprocess, sys
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h, units, v = rows[0], rows[1], rows[2]
want = ["gpu__time_duration.sum", "smsp__inst_executed.sum", "sm__inst_executed.avg.per_cycle_active",
        "sm__warps_active.avg.per_cycle_active", "launch__registers_per_thread", "launch__grid_size",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct",
        "l1tex__t_sector_hit_rate.pct", "launch__shared_mem_per_block_dynamic"]
for k in want:
    if k in h:
        i = h.index(k); print(f"{k:45s} {v[i]:>16s} {units[i]}")
for i, k in enumerate(h):
    if k.startswith("sm__inst_executed_pipe_") and k.endswith("avg.pct_of_peak_sustained_active"):
        try:
            if float(v[i]) > 3: print(f"{k:45s} {v[i]:>16s}")
        except ValueError: pass
for i, k in enumerate(h):
    if k.startswith("smsp__average_warp_latency_issue_stalled") or k.startswith("smsp__pcsamp_warps_issue_stalled"):
        pass
