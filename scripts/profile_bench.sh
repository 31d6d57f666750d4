#!/bin/bash
# ncu evidence for the benchmark (run under gpurun, one GPU):
#  1. launch list of a short bench run (per-launch device time, cold cache)
#  2. full captures of the f32 mover and deposit kernels (species 0 at step 5)
#  3. full capture of the bitwise-parity fused kernel
# Reports land in gpurun_out/; scripts/ncu_summarize.py writes profiles/.
set -x
R=${1:-r01}
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file gpurun_out/launches_$R.csv \
    python bench.py --steps 10 --warmup 0 --no-e2e --no-cpu --no-parity > gpurun_out/launches_$R.log 2>&1
for K in mover deposit; do
  ncu --set full --clock-control none --import-source on -k regex:${K}_kernel -s 20 -c 1 \
      -o gpurun_out/${K}_f32_$R python bench.py --steps 6 --warmup 0 --no-e2e --no-cpu --no-parity \
      > gpurun_out/${K}_f32_$R.log 2>&1
done
ncu --set full --clock-control none --import-source on -k regex:span_kernel -s 4 -c 1 \
    -o gpurun_out/span_parity_$R python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-parity --arith parity \
    > gpurun_out/span_parity_$R.log 2>&1
