#!/usr/bin/env bash
# quick GPU iteration: selected tests + one bench line
TAG=${1:-q}; shift || true
mkdir -p gpurun_out
timeout 600 python -m pytest -q -x "$@" > gpurun_out/${TAG}_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
tail -25 gpurun_out/${TAG}_pytest.log
if [ -z "$NOBENCH" ]; then
timeout 300 python bench.py --no-e2e --no-cpu --no-parity ${BENCHARGS} > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
echo "bench rc=$?"; tail -5 gpurun_out/${TAG}_bench.err
python - <<'PY' "$TAG"
import json, sys
try:
    d = json.load(open(f"gpurun_out/{sys.argv[1]}_bench.json"))
    print("value G/s", d["value"]/1e9, "ms/step", d["ms_per_step"])
    for k, v in d["roofline"]["kernels"].items():
        print(k, round(v["ms_per_launch"], 4), "ms", round(v["frac"], 3))
    print(d.get("extra"))
except Exception as e:
    print("bench parse failed", e)
PY
fi
