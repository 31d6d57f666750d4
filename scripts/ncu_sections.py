"""Executed warp-instructions per tile by line range of bp_f32.cu (sections
given as name:first-last,...), from an `ncu --page source --csv
--print-source sass,cuda` export.  usage: ncu_sections.py export.csv tiles spec"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
tiles = float(sys.argv[2])
secs = []
for part in sys.argv[3].split(","):
    name, rng = part.split(":")
    a, b = rng.split("-")
    secs.append((name, int(a), int(b)))
cur = None; fname = None; hdr = None
tot = {n: 0.0 for n, _, _ in secs}; tot["other"] = 0.0
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]; continue
    if len(r) >= 2 and r[0] == "Line No":
        hdr = r; continue
    if hdr is None or len(r) < 8: continue
    if r[0]:
        cur = (fname, int(r[0])); continue
    try: n = float(r[7])
    except ValueError: continue
    hit = "other"
    if cur and cur[0] == "bp_f32.cu":
        for name, a, b in secs:
            if a <= cur[1] <= b: hit = name; break
    tot[hit] += n
s = sum(tot.values())
for k, v in tot.items(): print(f"{k:12s} {v / tiles:8.1f} per tile  {100 * v / s:5.1f}%")
print(f"{'total':12s} {s / tiles:8.1f}")
