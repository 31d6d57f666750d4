"""Per-launch device time and warp instructions per 32-particle tile from an
ncu launch list (--metrics gpu__time_duration.sum,smsp__inst_executed.sum)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
tiles = float(sys.argv[2]) if len(sys.argv) > 2 else 65536000 / 32
i = [k for k, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[i]
ID, mi, vi = h.index("ID"), h.index("Metric Name"), h.index("Metric Value")
d = {}
for r in rows[i + 1:]:
    d.setdefault(int(r[ID]), {})[r[mi]] = float(r[vi].replace(",", ""))
for n, k in enumerate(sorted(d)):
    t = d[k]["gpu__time_duration.sum"] / 1e6
    ins = d[k].get("smsp__inst_executed.sum", 0) / tiles
    print(f"{n:3d} step {n // 4:2d} species {n % 4}  {t:6.3f} ms  {ins:6.0f} instr/tile")
