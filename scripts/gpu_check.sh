#!/usr/bin/env bash
# One gpurun session: the GPU test suite, smoke, and a default bench line.
# usage (here): gpurun --timeout 2400 -- 'bash scripts/gpu_check.sh TAG [pytest args...]'
TAG=${1:-run}; shift || true
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${TAG}_gpu.txt 2>&1
timeout 2000 python -m pytest tests -q -m gpu -x --durations=15 "$@" > gpurun_out/${TAG}_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/${TAG}_smoke.log
timeout 600 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
echo "bench rc=$?" >> gpurun_out/${TAG}_bench.err
tail -3 gpurun_out/${TAG}_pytest.log gpurun_out/${TAG}_smoke.log
