#!/bin/bash
# BASELINE.json configs beyond the headline, with clocks records (one GPU):
# C2 (2D GEM 256x128x1) bench lines per precision, the C5 sweep, the C4-style
# out-of-core run.  Outputs in gpurun_out/cfg_*.
mkdir -p gpurun_out
timeout 900 python -m pytest -q -x tests/test_gpu_init.py > gpurun_out/cfg_init_pytest.log 2>&1; tail -1 gpurun_out/cfg_init_pytest.log
for P in single mixed double; do
  timeout 600 python bench.py --cells 256,128,1 --precision $P --no-e2e --no-shuffled --cpu-seconds 4 \
      > gpurun_out/cfg_c2_$P.json 2> gpurun_out/cfg_c2_$P.err
  python scripts/bench_brief.py gpurun_out/cfg_c2_$P.json 2>/dev/null | head -1
done
timeout 1500 python scripts/sweep_c5.py --sizes 1e7,1e8,1e9 --steps 10 > gpurun_out/cfg_c5.jsonl 2> gpurun_out/cfg_c5.err
echo "c5 rc=$?"; tail -3 gpurun_out/cfg_c5.err
timeout 1500 python scripts/bench_out_of_core.py --particles 2e9 --budget-gb 8 --steps 2 > gpurun_out/cfg_c4.json 2> gpurun_out/cfg_c4.err
echo "c4 rc=$?"; tail -3 gpurun_out/cfg_c4.err; cat gpurun_out/cfg_c4.json | head -c 600
