#!/usr/bin/env bash
# One gpurun session: GPU tests, smoke, bench lines for both layouts.
# usage: gpurun --timeout 2700 -- 'bash scripts/gpu_session.sh TAG [pytest args...]'
TAG=${1:-run}; shift || true
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${TAG}_gpu.txt 2>&1
if [ -z "$NOTEST" ]; then
timeout 2000 python -m pytest tests -q -m gpu --durations=20 "$@" > gpurun_out/${TAG}_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/${TAG}_smoke.log
tail -3 gpurun_out/${TAG}_pytest.log gpurun_out/${TAG}_smoke.log
fi
for LAY in ${LAYOUTS:-bins flat}; do
timeout 600 python bench.py --layout $LAY $BENCHARGS > gpurun_out/${TAG}_bench_$LAY.json 2> gpurun_out/${TAG}_bench_$LAY.err
echo "bench $LAY rc=$?"; tail -3 gpurun_out/${TAG}_bench_$LAY.err
python scripts/bench_brief.py gpurun_out/${TAG}_bench_$LAY.json
done
