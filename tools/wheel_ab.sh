for lib in "$@"; do
  DEM_LIB_PATH=$lib timeout 600 python tools/wheel_bench.py --steps 20 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', round(d['ms_per_step'],2), round(d['stage_ms']['force+integrate'],2))"
done
