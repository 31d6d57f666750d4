#!/bin/bash
# Bench each prebuilt library variant in build_variants/ (dev tool).
cp paper_2008_04397_b200/libbp_b200.so /tmp/lib_orig.so
for v in build_variants/*.so; do
  cp $v paper_2008_04397_b200/libbp_b200.so
  echo "== $v"
  python bench.py --no-e2e --no-cpu --steps 20 2>/dev/null | python -c "
import json,sys
for ln in sys.stdin:
    if ln.startswith('{'):
        d=json.loads(ln); x=d['extra']
        print(f\"{d['value']/1e9:7.3f} G/s launch {d['roofline']['launch_ms']:.2f} ms parity {x.get('parity_arith',{}).get('value',0)/1e9:.3f} clk {d['clocks']}\")"
done
cp /tmp/lib_orig.so paper_2008_04397_b200/libbp_b200.so
