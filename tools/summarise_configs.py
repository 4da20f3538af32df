"""Table of the per-config bench lines and the C5 size curve (tools/config_sweep.sh output).

    python tools/summarise_configs.py r02
Writes profiles/<round>/configs.json (the JSON lines) and profiles/<round>/configs.md (the table).
"""
import glob
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def last_json(path):
    for line in reversed(open(path).read().splitlines()):
        if line.startswith("{"):
            return json.loads(line)
    return None


def main(rnd):
    src = os.path.join(ROOT, "gpurun_out", rnd, "configs")
    rows = {}
    for f in sorted(glob.glob(os.path.join(src, "bench_*.json"))):
        d = last_json(f)
        if d:
            rows[os.path.basename(f)[6:-5]] = d
    out = os.path.join(ROOT, "profiles", rnd)
    os.makedirs(out, exist_ok=True)
    json.dump(rows, open(os.path.join(out, "configs.json"), "w"), indent=1)
    lines = ["| run | workload | spheres | c (contacts/sphere) | ms/step | sphere-steps/s | e2e | dominant kernel | "
             "roofline frac | step frac (§8d) | oracle sphere-steps/s (1 core) |",
             "|---|---|---|---|---|---|---|---|---|---|---|"]
    for k, d in rows.items():
        cfg = d["config"]
        e2e = d.get("e2e") or {}
        cpu = d.get("cpu_baseline") or {}
        rf = d.get("roofline") or {}
        lines.append(f"| {k} | {cfg['workload']} | {cfg['spheres']:,} | {cfg['contacts_per_sphere']:.3f} | "
                     f"{d['ms_per_step']:.3f} | {d['value']:.3e} | {e2e.get('value', float('nan')):.3e} | "
                     f"{rf.get('kernel')} | {rf.get('frac', float('nan')):.3f} | "
                     f"{d['step_roofline']['frac']:.3f} | {cpu.get('value', float('nan')):.3e} |")
    stage = ["", "Stage times (ms/step, in-line profiled pass):", "",
             "| run | " + " | ".join(next(iter(rows.values()))["stage_ms"].keys()) + " |",
             "|---|" + "---|" * len(next(iter(rows.values()))["stage_ms"])]
    for k, d in rows.items():
        stage.append(f"| {k} | " + " | ".join(f"{v:.3f}" for v in d["stage_ms"].values()) + " |")
    text = "\n".join(lines + stage) + "\n"
    open(os.path.join(out, "configs.md"), "w").write(text)
    print(text)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r02")
