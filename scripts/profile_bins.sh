#!/bin/bash
# ncu evidence for the binned fast path (run under gpurun, one GPU):
#  launch list of a short bench run + full captures of mover_bins and
#  deposit_bins (species 0, third step).  Reports land in gpurun_out/.
R=${1:-r02}
mkdir -p gpurun_out
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file gpurun_out/launches_$R.csv \
    python bench.py --steps 6 --warmup 0 --no-e2e --no-cpu --no-parity > gpurun_out/launches_$R.log 2>&1
for K in mover_bins deposit_bins; do
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:$K -s 8 -c 1 \
      -o gpurun_out/${K}_$R python bench.py --steps 4 --warmup 0 --no-e2e --no-cpu --no-parity \
      > gpurun_out/${K}_$R.log 2>&1
done
python scripts/launch_summary.py gpurun_out/launches_$R.csv 2>&1 | head -40
