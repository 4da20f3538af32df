#!/bin/bash
# A/B stage timings of library variants on the bench workload: tools_ab.sh lib1.so lib2.so ...
for lib in "$@"; do
  DEM_LIB_PATH=$lib timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-variants 2>&1 | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', round(d['ms_per_step'],2), {k: round(v,2) for k,v in d['stage_ms'].items()})"
done
