#!/bin/bash
# compute-sanitizer suite (SURVEY §4 "Tooling"): memcheck, racecheck, synccheck, initcheck on the
# small cases of tools/sanitize_case.py.  Run under gpurun; logs in gpurun_out/$R/sanitize/.
#   tools/sanitize.sh r02
set -u
R=${1:-r02}
OUT=gpurun_out/$R/sanitize
mkdir -p "$OUT"
python -c "import paper_2307_03445_b200 as d; d.load_library()" || exit 1
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck synccheck initcheck racecheck; do
  for case in c1 deferred overlap mesh peer2 regrow empty; do
    extra=""
    [ "$tool" = memcheck ] && extra="--leak-check full"
    [ "$tool" = racecheck ] && extra="--racecheck-report all"
    timeout 900 $CS --tool $tool $extra --error-exitcode 99 python tools/sanitize_case.py $case \
      > "$OUT/${tool}_${case}.log" 2>&1
    echo "$tool $case rc=$?" | tee -a "$OUT/summary.txt"
  done
done
