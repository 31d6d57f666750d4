"""Key counters and stall shares of one ncu report: python ncu_brief.py REP [units]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(raw.splitlines()))
h, u, v = rows[0], rows[1], rows[2]
get = {k: (v[i], u[i]) for i, k in enumerate(h)}
for k in ["Kernel Name", "gpu__time_duration.sum", "smsp__inst_executed.sum",
          "sm__inst_executed.avg.per_cycle_active", "sm__warps_active.avg.per_cycle_active",
          "launch__registers_per_thread", "l1tex__t_sector_hit_rate.pct",
          "lts__t_sector_hit_rate.pct", "dram__bytes_read.sum", "dram__bytes_write.sum",
          "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
          "l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum",
          "l1tex__t_requests_pipe_lsu_mem_global_op_atom.sum",
          "lts__t_sectors_srcunit_tex_op_atom.sum", "launch__grid_size"]:
    if k in get:
        print(f"{k:55s} {get[k][0]} {get[k][1]}")
if len(sys.argv) > 2:
    n = float(get["smsp__inst_executed.sum"][0].replace(",", ""))
    print(f"warp instructions per unit: {n / float(sys.argv[2]):.1f}")
tot = float(get["smsp__pcsamp_sample_count"][0].replace(",", "")) if "smsp__pcsamp_sample_count" in get else 0
st = []
for k, (val, _) in get.items():
    if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("_not_issued"):
        try:
            st.append((float(val.replace(",", "")), k[len("smsp__pcsamp_warps_issue_stalled_"):]))
        except ValueError:
            pass
st.sort(reverse=True)
if tot:
    print("stalls:", ", ".join(f"{n}={100 * x / tot:.1f}%" for x, n in st[:9]))
