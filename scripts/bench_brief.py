"""One-screen summary of a bench.py JSON line (gpurun sessions)."""
import json
import sys

for path in sys.argv[1:]:
    try:
        d = json.loads(open(path).read().strip().splitlines()[-1])
    except Exception as e:  # noqa: BLE001
        print(path, "unparsable:", e)
        continue
    print(path, f"value {d['value'] / 1e9:.2f} G/s  ms/step {d['ms_per_step']:.3f}",
          "layout", d["config"].get("layout"), "clocks", d.get("clocks"))
    for k, v in d["roofline"]["kernels"].items():
        print(f"  {k:8s} {v['ms_per_launch']:.4f} ms/launch  frac {v['frac']:.3f}  "
              f"share {v['share_of_step']:.3f}")
    print("  fused_phase", d["roofline"]["fused_phase"])
    print("  extra", json.dumps(d.get("extra"))[:600])
    if d.get("e2e"):
        print("  e2e", d["e2e"]["value"] / 1e9, "G/s")
