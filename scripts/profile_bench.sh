#!/bin/bash
# ncu evidence for the benchmark (run under gpurun, one GPU):
#  1. launch list of a short bench run (per-launch device time, cold cache)
#  2. full capture of the fused kernel, fast arithmetic
#  3. full capture of the fused kernel, parity arithmetic
# Reports land in gpurun_out/; summaries are copied to profiles/ by hand.
set -x
R=${1:-r01}
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file gpurun_out/launches_$R.csv \
    python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-parity > gpurun_out/launches_$R.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:span_kernel -s 4 -c 1 \
    -o gpurun_out/span_fast_$R python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-parity \
    > gpurun_out/span_fast_$R.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:span_kernel -s 4 -c 1 \
    -o gpurun_out/span_parity_$R python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-parity --arith parity \
    > gpurun_out/span_parity_$R.log 2>&1
