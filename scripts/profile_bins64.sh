#!/bin/bash
# ncu evidence for the f64 binned path at C2 double (run under gpurun, one
# GPU): full captures of mover_bins64 / deposit_bins64 (species 0 of the
# third step) and a launch list.  Reports land in gpurun_out/.
#   usage: profile_bins64.sh TAG
R=${1:-r02c}
A="--cells 256,128,1 --precision double --no-e2e --no-cpu --no-parity --no-shuffled"
mkdir -p gpurun_out
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file gpurun_out/launches64_$R.csv \
    python bench.py --steps 4 --warmup 0 $A > gpurun_out/launches64_$R.log 2>&1
for K in mover_bins64 deposit_bins64; do
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:$K -s 8 -c 1 \
      -o gpurun_out/${K}_$R python bench.py --steps 4 --warmup 0 $A \
      > gpurun_out/${K}_$R.log 2>&1
done
