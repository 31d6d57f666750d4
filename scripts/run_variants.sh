#!/bin/bash
# on the GPU box: bench each build_variants/lib_<name>.so (short runs)
ROOT=$(cd "$(dirname "$0")/.." && pwd)
cp "$ROOT/paper_2008_04397_b200/libbp_b200.so" /tmp/lib_default.so
for f in "$ROOT"/build_variants/lib_*.so; do
  name=$(basename $f .so); name=${name#lib_}
  cp "$f" "$ROOT/paper_2008_04397_b200/libbp_b200.so"
  timeout 300 python "$ROOT/bench.py" --steps 8 --warmup 3 --no-e2e --no-cpu --no-parity $BENCHARGS > "$ROOT/gpurun_out/var_$name.json" 2> "$ROOT/gpurun_out/var_$name.err"
  python "$ROOT/scripts/bench_brief.py" "$ROOT/gpurun_out/var_$name.json" 2>/dev/null | head -3 | sed "s/^/[$name] /"
done
cp /tmp/lib_default.so "$ROOT/paper_2008_04397_b200/libbp_b200.so"
