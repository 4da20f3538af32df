"""Mesh contacts at the C5 scale (NEXT-3; the single-wheel test of P:441): a 0.25 m grousered
wheel mesh rolling with slip through the VIPER-scale bed (11.3M clumps / 34.7M spheres), timed
like bench.py (CUDA events, k = 1).  Writes gpurun_out/wheel_bench.json.

    python tools/wheel_bench.py [--steps K] [--warmup W]
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    a = ap.parse_args()
    import torch

    import paper_2307_03445_b200 as dem
    from workloads.beds import c5_bed
    from workloads.scenes import Mesh, mesh_wheel

    torch.cuda.set_device(0)
    s = c5_bed()
    R = 0.25
    cx, cy = 0.5 * (s.domain_lo[0] + s.domain_hi[0]), 0.5 * (s.domain_lo[1] + s.domain_hi[1])
    near = (np.abs(s.pos[:, 0] - cx) < 0.1) & (np.abs(s.pos[:, 1] - cy) < 0.1)
    top = float(s.pos[near, 2].max())
    wheel = mesh_wheel(R)
    # angular velocity 1.96 rad/s, slip (forward speed below omega R); sunk 2 cm
    w, v = 1.96, 0.3 * 1.96 * R
    s.meshes = [Mesh(wheel, 0, pos=(cx, cy, top + R - 0.02), vel=(v, 0.0, 0.0), omega=(0.0, w, 0.0))]
    g = dem.system_from_scene(s)
    g.dem_step(a.warmup)
    g.dem_set_profiling(True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(g.stream)
    g.dem_step(a.steps)
    e1.record(g.stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.steps
    st = g.dem_get_stats()
    stages = g.dem_get_stage_times()
    g.dem_set_profiling(False)
    m = g.dem_get_mesh(0)
    out = dict(workload="C5 bed + grousered wheel mesh (P:441 single-wheel slip)", spheres=st["n_spheres"],
               triangles=int(wheel.shape[0]), steps=a.steps, warmup=a.warmup, ms_per_step=ms,
               sphere_steps_per_s=st["n_spheres"] / (ms * 1e-3), contacts=st["n_contacts"],
               wheel_force_n=m["force"].tolist(), wheel_torque_nm=m["torque"].tolist(), stage_ms=stages,
               note="stage events between the kernels on the system stream (mesh pose in pose, mesh pairs in "
                    "bin_scatter, mesh finish in force)")
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    json.dump(out, open(os.path.join(ROOT, "gpurun_out", "wheel_bench.json"), "w"), indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
