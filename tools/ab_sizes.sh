#!/bin/bash
# Production-path ms/step of library variants at several sizes (C5, a C5/8 x-slab, C3), A B A B:
#   tools/ab_sizes.sh lib1.so lib2.so ...     (under gpurun)
for rep in 1 2; do
for lib in "$@"; do
  for run in "--config c5" "--config c5 --slab 0.125" "--config c5 --slab 0.0222" "--config c3"; do
    DEM_LIB_PATH=$lib timeout 600 python bench.py $run --steps ${STEPS:-200} --warmup ${WARM:-50} --prof-steps 5 \
      --no-cpu-baseline --no-e2e --no-variants 2>&1 | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', '$run', round(d['ms_per_step'],4), '%.3e' % d['value'])"
  done
done
done
