#!/bin/bash
# ncu evidence for the binned fast path (run under gpurun, one GPU):
#  launch list of a short bench run + full captures of the binned kernels
#  (species 0, third step).  Reports land in gpurun_out/.
#  usage: profile_bins.sh TAG [kernel regexes...]   (default: cycle_bins arrive_bins)
R=${1:-r02}; shift || true
KS=${@:-cycle_bins arrive_bins}
mkdir -p gpurun_out
if [ -z "$NOLAUNCH" ]; then
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file gpurun_out/launches_$R.csv \
    python bench.py --steps 6 --warmup 0 --no-e2e --no-cpu --no-parity > gpurun_out/launches_$R.log 2>&1
python scripts/launch_summary.py gpurun_out/launches_$R.csv 2>&1 | head -30
fi
for K in $KS; do
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:$K -s 8 -c 1 \
      -o gpurun_out/${K}_$R python bench.py --steps 4 --warmup 0 --no-e2e --no-cpu --no-parity \
      > gpurun_out/${K}_$R.log 2>&1
done
