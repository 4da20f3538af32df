#!/bin/bash
# Stage timings of the C5 bench at several bin edges (the contact set does not depend on them):
#   tools/cell_sweep.sh 0.0030 0.0033 0.0036 ...      (under gpurun)
for c in "$@"; do
  timeout 600 python bench.py --config ${CONFIG:-c5} --cell-size $c --steps ${STEPS:-30} --warmup ${WARM:-20} \
    --prof-steps ${STEPS:-30} --no-cpu-baseline --no-e2e --no-variants 2>&1 | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cell $c', round(d['ms_per_step'],3), d['config']['bin_inserts'], {k: round(v,3) for k,v in d['stage_ms'].items()})"
done
