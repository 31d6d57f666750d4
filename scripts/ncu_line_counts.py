"""Per-(file, line) executed warp-instruction counts from
`ncu --page source --csv --print-source sass,cuda`, normalised per unit.

    python scripts/ncu_line_counts.py mix.csv UNITS file.cuh:line [file:line ...]
"""
import csv
import sys


def load(path):
    hdr, cur, agg = None, None, {}
    for r in csv.reader(open(path)):
        if r and r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if len(r) > 3 and r[0] == "Line No":
            hdr = {h: i for i, h in enumerate(r)}
            width = len(r)
            continue
        if hdr and r and r[0].isdigit() and len(r) == width:
            try:
                n = float(r[hdr["Instructions Executed"]])
            except ValueError:
                n = 0.0
            agg[(cur, int(r[0]))] = (n, r[1])
    return agg


if __name__ == "__main__":
    agg = load(sys.argv[1])
    units = float(sys.argv[2])
    for spec in sys.argv[3:]:
        f, ln = spec.rsplit(":", 1)
        n, src = agg.get((f, int(ln)), (0.0, ""))
        print(f"{spec:>24s} {n / units:9.2f}  {src.strip()[:80]}")
