"""Per-kernel device times from an `ncu --metrics gpu__time_duration.sum --csv`
launch list: totals by kernel and the sequence of the named kernels."""
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1])))
names = sys.argv[2].split(",") if len(sys.argv) > 2 else ["mover", "deposit", "pack"]
h = None; seq = []
for r in rows:
    if "Kernel Name" in r: h = r; continue
    if h and len(r) == len(h):
        d = dict(zip(h, r))
        if d["Metric Name"] == "gpu__time_duration.sum":
            v = float(d["Metric Value"]) * (1e-3 if d["Metric Unit"] == "ns" else 1.0)
            seq.append((d["Kernel Name"], v))  # microseconds
tot = collections.defaultdict(float); cnt = collections.Counter()
for n, t in seq:
    k = n.split("(")[0][:60]; tot[k] += t; cnt[k] += 1
for k, t in sorted(tot.items(), key=lambda kv: -kv[1])[:15]:
    print(f"{t / 1e3:10.3f} ms  {cnt[k]:4d} x  {k}")
for nm in names:
    xs = [t for n, t in seq if nm in n]
    if xs: print(nm, "us:", " ".join(f"{x:.0f}" for x in xs))
