"""Summarise an ncu --set full report (selected metrics per kernel) as text / JSON."""
import csv
import io
import json
import subprocess
import sys

WANT = ["Duration", "DRAM Throughput", "Memory Throughput", "L1/TEX Cache Throughput", "L2 Cache Throughput",
        "L1/TEX Hit Rate", "L2 Hit Rate", "Compute (SM) Throughput", "Executed Ipc Active", "Achieved Occupancy",
        "Theoretical Occupancy", "Registers Per Thread", "Eligible Warps Per Scheduler", "No Eligible",
        "Warp Cycles Per Issued Instruction", "Dynamic Shared Memory Per Block", "Static Shared Memory Per Block"]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
       "l1tex__t_set_accesses_pipe_lsu_mem_global_op_atom.sum", "lts__t_sectors_op_atom.sum",
       "lts__t_sectors_op_red.sum", "sm__inst_executed_pipe_fp64.sum", "lts__t_bytes.sum",
       "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
       "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
       "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]


def summarise(rep):
    det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(det)))
    h = rows[0]
    ki, mi, ui, vi, ii = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Unit", "Metric Value", "ID"))
    out = {}
    for r in rows[1:]:
        if r[mi] in WANT:
            k = f"{r[ki].split('(')[0]}#{r[ii]}"
            out.setdefault(k, {})[r[mi]] = f"{r[vi]} {r[ui]}".strip()
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    hdr, units = rr[0], rr[1]
    for r in rr[2:]:
        k = f"{r[hdr.index('Kernel Name')].split('(')[0]}#{r[hdr.index('ID')]}"
        for m in RAW:
            if m in hdr:
                out.setdefault(k, {})[m] = f"{r[hdr.index(m)]} {units[hdr.index(m)]}".strip()
    return out


if __name__ == "__main__":
    s = summarise(sys.argv[1])
    if len(sys.argv) > 2:
        json.dump(s, open(sys.argv[2], "w"), indent=1)
    for k, v in s.items():
        print(k)
        for m, x in v.items():
            print(f"   {m:45s} {x}")
