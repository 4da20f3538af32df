#!/bin/bash
# Bench lines of every BASELINE config on one B200 and the per-rank size curve of the C5 bed
# (centred x-slabs: the share of one rank of a P-GPU slab decomposition, run as one system).
#   tools/config_sweep.sh r02          (under gpurun; summarise with tools/summarise_configs.py)
set -u
R=${1:-r02}
OUT=gpurun_out/$R/configs
mkdir -p "$OUT"
STEPS=${STEPS:-300}
WARM=${WARM:-50}
for c in c1 c3 c4; do
  timeout 900 python bench.py --config $c --steps $STEPS --warmup $WARM --no-variants > "$OUT/bench_$c.json" 2> "$OUT/bench_$c.err"
  echo "$c rc=$?"
done
for f in 0.5 0.25 0.125 0.0625 0.0222; do
  timeout 900 python bench.py --config c5 --slab $f --steps $STEPS --warmup $WARM --no-variants --no-e2e --no-cpu-baseline \
    > "$OUT/bench_c5_slab$f.json" 2> "$OUT/bench_c5_slab$f.err"
  echo "slab $f rc=$?"
done
