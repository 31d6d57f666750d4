"""Per-CUDA-source-line totals from `ncu --page source --csv --print-source sass,cuda`."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = None; out = []
for r in rows:
    if len(r) > 3 and r[0] == "Line No":
        hdr = r; continue
    if hdr and r and r[0] not in ("",) and len(r) == len(hdr) and r[0].isdigit():
        out.append(r)
ix = {h: i for i, h in enumerate(hdr)}
def f(r, k):
    try: return float(r[ix[k]])
    except Exception: return 0.0
ti = sum(f(r, "Instructions Executed") for r in out); ts = sum(f(r, "Warp Stall Sampling (All Samples)") for r in out)
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
key = sys.argv[3] if len(sys.argv) > 3 else "Warp Stall Sampling (All Samples)"
for r in sorted(out, key=lambda r: -f(r, key))[:n]:
    print(f"L{r[0]:>4s} instr {100*f(r,'Instructions Executed')/ti:5.2f}%  stall {100*f(r,'Warp Stall Sampling (All Samples)')/ts:5.2f}%  {r[1][:90]}")
