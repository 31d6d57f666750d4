#!/usr/bin/env bash
# Stage the reference package for the drop-in tests and the reference arm:
#   baseline/_ref/            pip install --target of /root/reference/pkg (batchpic)
#   baseline/_ref/ref_tests/  the reference's own test files (pkg/tests)
# Both are git-ignored (not product source) but travel to the GPU box with the
# gpurun snapshot; /root/reference itself does not exist there.
set -euo pipefail
ROOT=$(cd "$(dirname "$0")/.." && pwd)
REF=${REF:-/root/reference/pkg}
rm -rf /tmp/bp_refbuild "$ROOT/baseline/_ref"
cp -r "$REF" /tmp/bp_refbuild   # the build writes egg-info into its source tree
python -m pip install -q --no-index --no-build-isolation --no-deps \
  --find-links /opt/wheelhouse --target "$ROOT/baseline/_ref" /tmp/bp_refbuild
mkdir -p "$ROOT/baseline/_ref/ref_tests"
cp "$REF"/tests/*.py "$ROOT/baseline/_ref/ref_tests/"
echo "staged batchpic + $(ls "$ROOT/baseline/_ref/ref_tests" | wc -l) test files in baseline/_ref"
