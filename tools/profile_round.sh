#!/bin/bash
# Round evidence on the GPU box (run under gpurun): bench lines, the ncu launch list and one
# ncu --set full capture of every step kernel.  Summarise here with tools/summarise_round.py.
#   tools/profile_round.sh r01
set -u
R=${1:-r01}
OUT=gpurun_out/$R
mkdir -p "$OUT"
timeout 900 python bench.py > "$OUT/bench.json" 2> "$OUT/bench.err"
timeout 600 python bench.py --impl reference > "$OUT/bench_reference.json" 2> "$OUT/bench_reference.err"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file "$OUT/launches.csv" \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-variants > "$OUT/launches.log" 2>&1
# one launch of each step kernel, after the warm-up steps
timeout 1500 ncu --set full --import-source on --clock-control none \
  -k regex:"k_pose_count|k_bin_scatter|k_pairs|k_rows_finish|k_force_integrate" --launch-skip 15 --launch-count 5 \
  -o "$OUT/full" python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-variants > "$OUT/full.log" 2>&1
# measured FP64 FMA peak (SURVEY §8d FP64 check)
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/fp64_peak tools/fp64_peak.cu && /tmp/fp64_peak > "$OUT/fp64_peak.json"
tail -c 300 "$OUT/bench.json"
