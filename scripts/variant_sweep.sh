#!/bin/bash
# bench kernel times per BP_BINS_VARIANT value (args)
for v in "$@"; do
  BP_BINS_VARIANT=$v timeout 200 python bench.py --steps 6 --warmup 3 --no-e2e --no-cpu --no-parity > gpurun_out/var_$v.json 2>/dev/null
  python - "$v" <<'PY'
import json, sys
v = sys.argv[1]
try:
    d = json.load(open(f"gpurun_out/var_{v}.json"))
    k = d["roofline"]["kernels"]
    print(f"variant {v:>3}: {d['value']/1e9:6.2f} G/s  step {d['ms_per_step']:6.2f} ms  mover {k['mover']['ms_per_launch']:.4f}  deposit {k['deposit']['ms_per_launch']:.4f}  phase3 {d['extra']['phase3_kernel_ms_per_step']:.2f}")
except Exception as e:
    print(v, "failed", e)
PY
done
