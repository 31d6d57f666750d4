"""Summarise an `ncu --page source --csv --print-source sass` export:
instructions executed and stall samples per opcode, top stall sites."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
data = [r for r in rows[2:] if len(r) == len(hdr)]
def f(r, k):
    try: return float(r[ix[k]].replace(',', ''))
    except Exception: return 0.0
by_op = collections.Counter(); st_op = collections.Counter()
tot_i = sum(f(r, "Instructions Executed") for r in data)
tot_s = sum(f(r, "Warp Stall Sampling (All Samples)") for r in data)
for r in data:
    toks = r[ix["Source"]].split()
    if not toks: continue
    op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
    op = op.split(".")[0]
    by_op[op] += f(r, "Instructions Executed")
    st_op[op] += f(r, "Warp Stall Sampling (All Samples)")
print(f"total warp-instructions {tot_i:.4g}, stall samples {tot_s:.4g}")
print("opcode            instr%   stall%")
for op, v in by_op.most_common(25):
    print(f"{op:16s} {100*v/tot_i:6.2f}  {100*st_op[op]/max(tot_s,1):6.2f}")
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
agg = {h: sum(f(r, h) for r in data) for h in stalls}
print("stall reasons:", ", ".join(f"{k[6:]}={100*v/max(tot_s,1):.1f}%" for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:8]))
top = sorted(data, key=lambda r: -f(r, "Warp Stall Sampling (All Samples)"))[:int(sys.argv[2]) if len(sys.argv) > 2 else 15]
for r in top:
    print(f"{r[ix['Address']]:>8s} {100*f(r,'Warp Stall Sampling (All Samples)')/tot_s:5.2f}% {r[ix['Source']][:70]}")
