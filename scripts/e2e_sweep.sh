#!/bin/bash
# Host-buffer e2e leg (bp_fused_span_host) at several batch sizes (one GPU):
#   gpurun -- 'bash scripts/e2e_sweep.sh TAG'
TAG=${1:-e2e}
mkdir -p gpurun_out
for B in ${BATCHES:-1048576 2097152 4194304 8388608}; do
  BP_HOST_BATCH=$B timeout 600 python bench.py --steps 3 --warmup 3 --e2e-steps 4 --no-cpu \
      --no-parity --no-shuffled --no-c2-double --no-streams-leg \
      > gpurun_out/${TAG}_b$B.json 2> gpurun_out/${TAG}_b$B.err
  python - gpurun_out/${TAG}_b$B.json $B <<'EOF'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print("batch", sys.argv[2], "e2e", d["e2e"]["value"], "value", d["value"])
EOF
done
