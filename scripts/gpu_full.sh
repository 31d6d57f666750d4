#!/bin/bash
# One full evidence session: GPU tests, smoke, bench lines (default = binned
# layout, and the flat layout), racecheck, ncu profile.
TAG=${1:-full}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${TAG}_gpu.txt 2>&1
timeout 2400 python -m pytest tests -q -m gpu --durations=25 > gpurun_out/${TAG}_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log; tail -3 gpurun_out/${TAG}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/${TAG}_smoke.log; tail -2 gpurun_out/${TAG}_smoke.log
timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
echo "bench rc=$?"; python scripts/bench_brief.py gpurun_out/${TAG}_bench.json
timeout 600 python bench.py --layout flat --no-e2e --no-cpu --no-shuffled > gpurun_out/${TAG}_bench_flat.json 2> gpurun_out/${TAG}_bench_flat.err
python scripts/bench_brief.py gpurun_out/${TAG}_bench_flat.json | head -4
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${TAG}_bench_ref.json 2> gpurun_out/${TAG}_bench_ref.err
if [ -z "$NOPROF" ]; then
BP_TMA_STREAM=1 timeout 1200 compute-sanitizer --tool racecheck --print-limit 20 \
    python scripts/debug/sanitize_driver.py > gpurun_out/sanitize_racecheck.txt 2>&1
tail -2 gpurun_out/sanitize_racecheck.txt
bash scripts/profile_r02.sh r02b
fi
