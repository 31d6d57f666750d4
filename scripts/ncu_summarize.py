"""Summarise the profile_bench.sh captures into profiles/: ncu_summary_<R>.json
(counters per kernel), <kernel>_<R>_sass_summary.txt, <kernel>_<R>_details.csv,
and the launch list."""
import csv, json, os, shutil, subprocess, sys
R = sys.argv[1] if len(sys.argv) > 1 else "r01"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G, P = os.path.join(ROOT, "gpurun_out"), os.path.join(ROOT, "profiles")
WANT = {"gpu__time_duration.sum": "gpu_time_ms_under_ncu", "smsp__inst_executed.sum": "issued_warp_instructions",
        "sm__inst_executed.avg.per_cycle_active": "ipc_active", "sm__warps_active.avg.per_cycle_active": "achieved_warps_per_sm",
        "launch__registers_per_thread": "registers_per_thread", "l1tex__t_sector_hit_rate.pct": "l1_hit_pct",
        "lts__t_sector_hit_rate.pct": "l2_hit_pct", "dram__bytes_read.sum": "dram_bytes_read_per_launch",
        "dram__bytes_write.sum": "dram_bytes_write_per_launch", "launch__grid_size": "grid",
        "launch__shared_mem_per_block_dynamic": "smem_per_block_bytes"}
SCALE = {"ms": 1.0, "us": 1e-3, "ns": 1e-6, "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
out_path = os.path.join(P, f"ncu_summary_{R}.json")
summary = json.load(open(out_path)) if os.path.exists(out_path) else {}
# key=report pairs after the round tag (reports gpurun_out/<report>.ncu-rep);
# default: the round-1 captures of scripts/profile_bench.sh
PAIRS = [a.split("=", 1) for a in sys.argv[2:]] or [
    ("mover", f"mover_f32_{R}"), ("deposit", f"deposit_f32_{R}"),
    ("span_kernel_parity", f"span_parity_{R}")]
for key, rep in PAIRS:
    path = os.path.join(G, rep + ".ncu-rep")
    if not os.path.exists(path):
        continue
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    h, u, v = rows[0], rows[1], rows[2]
    d = {"kernel": v[h.index("Kernel Name")] if "Kernel Name" in h else key,
         "capture": f"gpurun_out/{rep}.ncu-rep (round {R})"}
    for m, name in WANT.items():
        if m in h:
            i = h.index(m)
            try:
                val = float(v[i].replace(",", ""))
            except ValueError:
                continue
            d[name] = val * SCALE.get(u[i], 1.0) if u[i] in SCALE else val
    if "dram_bytes_read_per_launch" in d:
        d["dram_bytes_per_launch"] = d["dram_bytes_read_per_launch"] + d.get("dram_bytes_write_per_launch", 0.0)
    summary[key] = d
    det = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    open(os.path.join(P, f"{rep}_details.csv"), "w").write(det)
    src = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    tmp = os.path.join(G, rep + "_sass.csv"); open(tmp, "w").write(src)
    txt = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "ncu_sass_summary.py"), tmp, "20"],
                         capture_output=True, text=True).stdout
    open(os.path.join(P, f"{rep}_sass_summary.txt"), "w").write(txt)
json.dump(summary, open(out_path, "w"), indent=1)
lp = os.path.join(G, f"launches_{R}.csv")
if os.path.exists(lp):
    shutil.copy(lp, os.path.join(P, f"{R}_launches.csv"))
print(json.dumps(summary, indent=1))
