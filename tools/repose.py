"""NEXT-4: repose angle of the DS material poured through a funnel.

Runs on the GPU (the oracle is far too slow for ~1e6 steps of 30k spheres): the scaled-down P:277
recipe of workloads/repose.py, deferred contact-set rebuild (k = 10) with a margin for
the fall speed, until the pile is at rest; then the free-surface angle.  Writes
gpurun_out/repose.json.

    python tools/repose.py [--max-steps N] [--chunk N]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--max-steps", type=int, default=1_500_000)
    ap.add_argument("--chunk", type=int, default=50_000)
    ap.add_argument("--vmax", type=float, default=4.0)
    ap.add_argument("--cd-every", type=int, default=10)
    ap.add_argument("--copies", type=int, default=4)
    ap.add_argument("--funnel", default="0.07,0.03,0.05,0.08", help="r_top,r_open,height,z_bottom [m]")
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "repose.json"))
    a = ap.parse_args()
    import torch

    import paper_2307_03445_b200 as dem
    from workloads.repose import pile_angle, repose_scene

    torch.cuda.set_device(0)
    rt, ro, fh, fz = (float(x) for x in a.funnel.split(","))
    s = repose_scene(copies=a.copies, r_top=rt, r_open=ro, funnel_h=fh, funnel_z=fz)
    k = a.cd_every
    margin = 2.0 * a.vmax * s.h * k
    g = dem.system_from_scene(s, margin=margin, cd_every=k)
    rb = np.array([t.bounding_radius for t in s.templates])[s.tid]
    mass = np.array([t.mass for t in s.templates])[s.tid]
    log = []
    t0 = time.time()
    steps = 0
    rest = 0
    while steps < a.max_steps:
        g.dem_step(a.chunk)
        steps += a.chunk
        st = g.dem_get_state()
        order = np.argsort(st["gid"])
        v = st["vel"][order]
        z = st["pos"][order][:, 2]
        ke = float(0.5 * np.sum(mass * np.sum(v * v, axis=1)))
        in_funnel = int(np.sum(z > s.meshes[0].pos[2]))
        vmax = float(np.abs(v).max())
        log.append(dict(step=steps, t_s=steps * s.h, ke_j=ke, in_funnel=in_funnel, vmax=vmax,
                        wall_s=time.time() - t0))
        print(json.dumps(log[-1]), flush=True)
        rest = rest + 1 if (in_funnel < 0.01 * s.n_clumps and vmax < 0.05) else 0
        if rest >= 3:
            break
    st = g.dem_get_state()
    order = np.argsort(st["gid"])
    pos = st["pos"][order]
    res = pile_angle(pos, rb, z_max=s.meshes[0].pos[2])
    wall = time.time() - t0
    out = dict(scene=s.name, clumps=s.n_clumps, spheres=s.n_spheres, steps=steps, sim_time_s=steps * s.h,
               h=s.h, cd_every=k, margin_m=margin, gpu_wall_s=wall,
               sphere_steps_per_s=s.n_spheres * steps / wall, paper_angle_deg=30.0, **res, log=log)
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    json.dump(out, open(a.out, "w"), indent=1)
    print(json.dumps({k_: v_ for k_, v_ in out.items() if k_ not in ("profile", "log")}))


if __name__ == "__main__":
    main()
