#!/bin/bash
# build libbp_b200.so variants into build_variants/lib_<name>.so
#   usage: build_variants.sh name1="-DFOO=1 -DBAR=2" name2="..."
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
mkdir -p "$ROOT/build_variants"
for spec in "$@"; do
  name=${spec%%=*}; flags=${spec#*=}
  make -s -C "$ROOT/paper_2008_04397_b200/csrc" clean >/dev/null
  make -s -C "$ROOT/paper_2008_04397_b200/csrc" -j8 NVCC="nvcc $flags" >/dev/null 2>&1 || { echo "build $name failed"; exit 1; }
  cp "$ROOT/paper_2008_04397_b200/libbp_b200.so" "$ROOT/build_variants/lib_$name.so"
  grep -A2 "${KGREP:-mover_bins}" "$ROOT/paper_2008_04397_b200/csrc/bp_bins.ptxas.txt" | grep Used | head -1 | sed "s/^/$name: /"
done
make -s -C "$ROOT/paper_2008_04397_b200/csrc" clean >/dev/null
make -s -C "$ROOT/paper_2008_04397_b200/csrc" -j8 >/dev/null 2>&1
