#!/bin/bash
# ncu evidence for round 2 (one GPU; reports in gpurun_out/, summarised by
#   python scripts/ncu_summarize.py r02 mover_bins=mover_bins_r02 ...):
#  1. launch list of a short default bench run (binned layout; per-launch
#     device time and DRAM bytes, cold cache, serialised)
#  2. full captures of the binned kernels (species 0, third step) and of the
#     flat split kernels (species 0 at step 5 of the sort period)
R=${1:-r02b}
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file gpurun_out/launches_$R.csv \
    python bench.py --steps 6 --warmup 0 --no-e2e --no-cpu --no-parity --no-shuffled --no-c2-double --no-streams-leg > gpurun_out/launches_$R.log 2>&1
# deposit_bins is two template kernels (the misplaced-check variant returns at
# once when the mover found none): select the common one by mangled name
for K in mover_bins deposit_binsILb0 migrate_bins; do
  timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base mangled \
      -k regex:$K -s 8 -c 1 \
      -o gpurun_out/${K}_$R python bench.py --steps 4 --warmup 0 --no-e2e --no-cpu --no-parity --no-shuffled \
      --no-c2-double --no-streams-leg \
      > gpurun_out/${K}_$R.log 2>&1
done
for K in mover deposit; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:${K}_kernel -s 20 -c 1 \
      -o gpurun_out/${K}_f32_$R python bench.py --layout flat --steps 6 --warmup 0 --no-e2e --no-cpu \
      --no-parity --no-shuffled --no-c2-double --no-streams-leg > gpurun_out/${K}_f32_$R.log 2>&1
done
ls -la gpurun_out/*_$R.ncu-rep
