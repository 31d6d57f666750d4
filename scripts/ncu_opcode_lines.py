"""For a given opcode, which CUDA source lines execute it (sass,cuda export)."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
want = sys.argv[2]
hdr = None; cur = None; cnt = collections.Counter(); tot = 0
for r in rows:
    if len(r) > 3 and r[0] == "Line No":
        hdr = r; ix = {h: i for i, h in enumerate(hdr)}; continue
    if not hdr or len(r) != len(hdr): continue
    if r[0].isdigit():
        cur = f"L{r[0]} {r[1][:70]}"; continue
    src = r[3].split()
    if not src: continue
    op = src[1] if src[0].startswith("@") and len(src) > 1 else src[0]
    try: n = float(r[ix["Instructions Executed"]])
    except: n = 0
    if op.split(".")[0] == want:
        cnt[cur] += n; tot += n
for k, v in cnt.most_common(15): print(f"{100*v/max(tot,1):5.1f}% {k}")
