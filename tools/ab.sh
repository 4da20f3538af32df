#!/bin/bash
# A/B stage timings of library variants on the bench workload, interleaved twice (A B A B):
#   tools/ab.sh lib1.so lib2.so ...        (CONFIG=c4 tools/ab.sh ... for another bed)
CONFIG=${CONFIG:-c5}
for rep in 1 2; do
for lib in "$@"; do
  DEM_LIB_PATH=$lib timeout 600 python bench.py --config $CONFIG --steps ${STEPS:-30} --warmup ${WARM:-20} \
    --prof-steps ${STEPS:-30} --no-cpu-baseline --no-e2e --no-variants 2>&1 | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['stage_ms'].items()})"
done
done
