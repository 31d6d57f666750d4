"""Per-source-line executed counts of one SASS opcode prefix, from an
`ncu --page source --csv --print-source sass,cuda` export.
usage: ncu_opcode_by_line.py export.csv OPCODE_PREFIX [tiles]"""
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1])))
pref = sys.argv[2]
tiles = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
cur = None; fname = None; hdr = None
cnt = collections.Counter(); src = {}
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]; continue
    if len(r) >= 2 and r[0] == "Line No":
        hdr = r; continue
    if hdr is None or len(r) < 8:
        continue
    if r[0]:
        cur = (fname, r[0]); src[cur] = r[1][:70]; continue
    sass = r[3].split()
    if not sass: continue
    op = sass[1] if sass[0].startswith("@") and len(sass) > 1 else sass[0]
    if op.startswith(pref):
        try: n = float(r[7])
        except ValueError: n = 0.0
        cnt[cur] += n
for k, v in cnt.most_common(20):
    print(f"{k[0]}:{k[1]:>4s} {v / tiles:8.1f}  {src.get(k, '')}")
