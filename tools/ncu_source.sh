#!/bin/bash
# Source-level (SASS + CUDA line) capture of one launch each of k_pairs and k_force_integrate on
# the bench bed (under gpurun); read here with
#   ncu -i gpurun_out/<tag>/src.ncu-rep --page source --csv --print-source sass,cuda
#   tools/ncu_source.sh <tag> [extra bench args]
set -u
T=${1:-src}
shift || true
OUT=gpurun_out/$T
mkdir -p "$OUT"
timeout 1200 ncu --set full --import-source on --clock-control none \
  -k regex:"k_pairs|k_force_integrate" --launch-skip 6 --launch-count 2 -o "$OUT/src" -f \
  python bench.py --steps 1 --warmup 3 --prof-steps 2 --no-cpu-baseline --no-e2e --no-variants "$@" > "$OUT/src.log" 2>&1
echo "ncu rc=$?"
ls -la "$OUT"
