#!/bin/bash
# Repeatable perf matrix under gpurun: GPU state first, then bench variants.
nvidia-smi --query-gpu=name,clocks.sm,clocks.mem,clocks.max.sm,power.draw,temperature.gpu,utilization.gpu --format=csv
nvidia-smi --query-compute-apps=pid,name,used_memory --format=csv
summ() { python -c "
import json,sys
for ln in sys.stdin:
    ln=ln.strip()
    if not ln.startswith('{'): continue
    d=json.loads(ln); x=d.get('extra',{})
    print(f\"{sys.argv[1]:28s} {d['value']/1e9:7.3f} G/s  step {d['ms_per_step']:7.2f} ms  launch {d['roofline']['launch_ms']:6.2f} ms  sort {x.get('sort_ms_per_sort',0):6.1f} ms  clk {d['clocks'].get('sm_mhz')} pw {d['clocks'].get('power_w_max')} {d['clocks'].get('reasons')} parity {x.get('parity_arith',{}).get('value',0)/1e9:.3f}\")
" "$1"; }
for rep in 1 2; do
  python bench.py --no-e2e --no-cpu --steps 20 "$@" 2>/dev/null | summ "fast rep$rep"
done
python bench.py --no-e2e --no-cpu --no-parity --arith parity --steps 10 "$@" 2>/dev/null | summ "parity"
