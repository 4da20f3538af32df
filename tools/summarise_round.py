"""Summarise a round's GPU evidence (tools/profile_round.sh) into profiles/<round>/.

  python tools/summarise_round.py r01

Writes: bench_c5.json, bench_reference_oracle.json (the JSON lines), ncu_launches_c5.csv and
ncu_launches_c5_summary.txt (per-kernel launch times and share of the step from the ncu launch
list), ncu_full.json / ncu_full.txt (selected metrics of the --set full capture), and
profiles/ncu_traffic.json (DRAM bytes per launch of each bench stage, read by bench.py as
roofline.traffic).
"""
import csv
import io
import json
import os
import shutil
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "profiles"))
from ncu_summary import summarise  # noqa: E402

STAGE_OF = {"k_pose_count": "pose+bin_count", "k_bin_scatter": "bin_scatter", "k_pairs": "pairs",
            "k_rows_finish": "rows_finish", "k_force_integrate": "force+integrate"}


def last_json_line(path):
    for line in reversed(open(path).read().splitlines()):
        if line.startswith("{"):
            return json.loads(line)
    raise ValueError(f"no JSON line in {path}")


def launch_summary(csv_path):
    text = open(csv_path).read()
    text = text[text.index('"ID"'):]
    rows = list(csv.DictReader(io.StringIO(text)))
    per = {}
    for r in rows:
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        k = r["Kernel Name"].split("(")[0].replace("void ", "")
        per.setdefault(k, []).append(float(r["Metric Value"]) * (1e-6 if r["Metric Unit"] == "ns" else 1e-3))
    total = sum(sum(v) for v in per.values())
    lines = ["ncu --metrics gpu__time_duration.sum --clock-control none, python bench.py --steps 2 --warmup 3 "
             "(C5 bed, 34.7M spheres)",
             "cold-cache, serialised launches: compare shares with bench.py stage_ms, not absolutes"]
    for k, v in per.items():
        lines.append(f"{k:28s} launches={len(v):3d} mean={sum(v) / len(v):.3f} ms  share_of_step={100 * sum(v) / total:.1f}%")
    return "\n".join(lines) + "\n"


def atomics_summary(csv_path):
    """Per-kernel means of the explicitly requested atomic / L2 / DRAM counters (north_star)."""
    text = open(csv_path).read()
    text = text[text.index('"ID"'):]
    rows = list(csv.DictReader(io.StringIO(text)))
    per = {}
    for r in rows:
        k = r["Kernel Name"].split("(")[0].replace("void ", "")
        try:
            v = float(r["Metric Value"].replace(",", ""))
        except ValueError:
            continue
        per.setdefault(k, {}).setdefault(f"{r['Metric Name']} [{r['Metric Unit']}]", []).append(v)
    out = {k: {m: sum(v) / len(v) for m, v in ms.items()} for k, ms in per.items()}
    lines = ["ncu --clock-control none --metrics <atomic, L2 and DRAM counters> (C5 bed, mean per launch)"]
    for k, ms in out.items():
        lines.append(k)
        for m, v in sorted(ms.items()):
            lines.append(f"   {m:75s} {v:.6g}")
    return out, "\n".join(lines) + "\n"


def main(rnd):
    src = os.path.join(ROOT, "gpurun_out", rnd)
    dst = os.path.join(ROOT, "profiles", rnd)
    os.makedirs(dst, exist_ok=True)
    json.dump(last_json_line(os.path.join(src, "bench.json")), open(os.path.join(dst, "bench_c5.json"), "w"))
    ref = os.path.join(src, "bench_reference.json")
    if os.path.exists(ref):
        json.dump(last_json_line(ref), open(os.path.join(dst, "bench_reference_oracle.json"), "w"))
    fp = os.path.join(src, "fp64_peak.json")
    if os.path.exists(fp):
        shutil.copy(fp, os.path.join(dst, "fp64_peak.json"))
    lc = os.path.join(src, "launches.csv")
    if os.path.exists(lc):
        shutil.copy(lc, os.path.join(dst, "ncu_launches_c5.csv"))
        open(os.path.join(dst, "ncu_launches_c5_summary.txt"), "w").write(launch_summary(lc))
    at = os.path.join(src, "atomics.csv")
    if os.path.exists(at):
        d, txt = atomics_summary(at)
        json.dump(d, open(os.path.join(dst, "ncu_atomics.json"), "w"), indent=1)
        open(os.path.join(dst, "ncu_atomics.txt"), "w").write(txt)
    rep = os.path.join(src, "full.ncu-rep")
    if os.path.exists(rep):
        s = summarise(rep)
        json.dump(s, open(os.path.join(dst, "ncu_full.json"), "w"), indent=1)
        with open(os.path.join(dst, "ncu_full.txt"), "w") as f:
            for k, v in s.items():
                f.write(k + "\n")
                for m, x in v.items():
                    f.write(f"   {m:45s} {x}\n")
        traffic = {}
        for k, v in s.items():
            name = k.split("#")[0].split("::")[-1].replace("void ", "").split("<")[0].strip()
            if name in STAGE_OF and "dram__bytes_read.sum" in v:
                def gb(x):
                    val, unit = x.split()
                    return float(val) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[unit]
                traffic[STAGE_OF[name]] = gb(v["dram__bytes_read.sum"]) + gb(v["dram__bytes_write.sum"])
        path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        allt = json.load(open(path)) if os.path.exists(path) else {}
        allt["c5"] = traffic
        allt["_source"] = f"profiles/{rnd}/ncu_full.json (ncu --set full, one launch per kernel, C5 bed)"
        json.dump(allt, open(path, "w"), indent=1)
    print("wrote", dst)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r01")
