#!/bin/bash
# Round evidence on the GPU box (run under gpurun): bench lines, the ncu launch list, one
# ncu --set full capture of every step kernel, and the north_star atomic / L2 counters.
# Summarise here with tools/summarise_round.py.
#   tools/profile_round.sh r02 [quick]
set -u
R=${1:-r02}
OUT=gpurun_out/$R
mkdir -p "$OUT"
if [ "${2:-}" != quick ]; then
  timeout 1200 python bench.py > "$OUT/bench.json" 2> "$OUT/bench.err"
  timeout 600 python bench.py --impl reference > "$OUT/bench_reference.json" 2> "$OUT/bench_reference.err"
fi
NCUB="python bench.py --steps 2 --warmup 3 --prof-steps 2 --no-cpu-baseline --no-e2e --no-variants"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file "$OUT/launches.csv" \
  $NCUB > "$OUT/launches.log" 2>&1
# one launch of each step kernel, after the warm-up steps (graph launches are not profiled
# kernel by kernel, so the capture runs in the in-line stage pass: --steps 1 --prof-steps 2)
timeout 1500 ncu --set full --import-source on --clock-control none \
  -k regex:"k_pose_count|k_bin_scatter|k_pairs|k_rows_finish|k_force_integrate" --launch-skip 15 --launch-count 5 \
  -o "$OUT/full" -f $NCUB > "$OUT/full.log" 2>&1
# atomics and L2 traffic (north_star: "achieved HBM GB/s ... plus atomic and L2 throughput")
timeout 900 ncu --clock-control none --csv --log-file "$OUT/atomics.csv" \
  -k regex:"k_pose_count|k_bin_scatter|k_pairs|k_rows_finish|k_force_integrate|excl_scan" --launch-skip 20 --launch-count 10 \
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,lts__t_sectors_op_atom.sum,lts__t_sectors_op_red.sum,l1tex__t_set_accesses_pipe_lsu_mem_global_op_atom.sum,l1tex__t_set_accesses_pipe_lsu_mem_global_op_red.sum,l1tex__t_requests_pipe_lsu_mem_global_op_atom.sum,lts__t_sectors_srcunit_tex_op_atom.sum,smsp__inst_executed.sum,lts__throughput.avg.pct_of_peak_sustained_elapsed \
  $NCUB > "$OUT/atomics.log" 2>&1
if [ "${2:-}" != quick ]; then
  nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/fp64_peak tools/fp64_peak.cu && /tmp/fp64_peak > "$OUT/fp64_peak.json"
  tail -c 300 "$OUT/bench.json"
fi
