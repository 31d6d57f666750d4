"""Per-unit executed warp instructions of one kernel capture, deduplicated by
SASS address (the mixed source export lists an inlined instruction under
every source file it maps to), by opcode and by bp_split.cu line.

    ncu -i REP --page source --csv --print-source sass,cuda > mix.csv
    python scripts/ncu_tile_breakdown.py mix.csv UNITS [top]
"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
units = float(sys.argv[2])
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
hdr, fname, cur = None, None, None
seen = {}
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) >= 2 and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8:
        continue
    if r[0]:
        cur = (fname, int(r[0]), r[1][:80])
        continue
    sass = r[3].split()
    if not sass:
        continue
    op = sass[1] if sass[0].startswith("@") and len(sass) > 1 else sass[0]
    try:
        n = float(r[7])
    except ValueError:
        n = 0.0
    # keep the bp_*.cu attribution when an address appears more than once
    if r[2] not in seen or (cur[0].startswith("bp_") and not seen[r[2]][1][0].startswith("bp_")):
        seen[r[2]] = (n, cur, op.split(".")[0])
tot = sum(v[0] for v in seen.values())
print(f"warp instructions per unit: {tot / units:.1f}")
byop, byline = collections.Counter(), collections.Counter()
for n, cur, op in seen.values():
    byop[op] += n
    byline[cur] += n
print("by opcode:", ", ".join(f"{k} {v / units:.1f}" for k, v in byop.most_common(16)))
for (f, l, s), v in byline.most_common(top):
    print(f"{f[:14]}:{l:<5d} {v / units:7.1f}  {s}")
