"""Write the settled DS base patch used to tile the C4/C5 beds — calls ONLY `oracle/`.

Recipe (DESIGN.md §"Input recipe"): spawn DS clumps (Table-1 number
fractions) by exact-geometry RSA in a 30 x 30 mm column at ~27% solid fraction,
all moving down at 1 m/s, and let them settle under gravity in a 5-wall box with
the CPU oracle at h = 1e-6 s (material M0) until the fastest clump is slower than
`--vstop`, then (``--resume ... --frictionless-sides``) settle it further with the four side walls
frictionless, because the beds replace those walls by the patch's mirror images, whose contacts
carry no tangential force.  The result is a dense settled patch that `workloads.beds.tiled_bed`
copy-pastes into the multi-million-clump benchmark beds.  The committed patch:
140,000 steps in the 5-wall box, then 100,000 steps with frictionless side walls (0.24 s of
settling; mean speed 0.8 mm/s, 1.09 contacts per sphere).  Since the state is produced by the oracle,
no benchmark or parity input ever comes from the CUDA path.

    python -m workloads.make_patch --out workloads/data/ds_patch_30mm.npz
"""
from __future__ import annotations

import argparse
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import oracle  # noqa: E402
from workloads.scenes import rsa_bed_exact, save_scene  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="workloads/data/ds_patch_30mm.npz")
    ap.add_argument("--seed", type=int, default=2307)
    ap.add_argument("--side", type=float, default=0.03)
    ap.add_argument("--depth", type=float, default=0.15, help="target settled depth [m]")
    ap.add_argument("--fraction", type=float, default=0.27)
    ap.add_argument("--density", type=float, default=3.05e7, help="settled clumps per m^3 (P:233-234)")
    ap.add_argument("--vz", type=float, default=-1.0)
    ap.add_argument("--vstop", type=float, default=0.02)
    ap.add_argument("--max-steps", type=int, default=400000)
    ap.add_argument("--chunk", type=int, default=2000)
    ap.add_argument("--resume", default=None,
                    help="continue settling a saved patch (its state, no history) instead of spawning")
    ap.add_argument("--frictionless-sides", action="store_true",
                    help="make the four side walls frictionless (mu = 0): the beds replace them by mirror "
                         "images, whose contacts carry no tangential force")
    a = ap.parse_args()
    import workloads as w

    t0 = time.time()
    if a.resume:
        from workloads.scenes import load_scene

        s = load_scene(a.resume)
        steps = int(s.name.rsplit("-", 1)[-1]) if s.name.rsplit("-", 1)[-1].isdigit() else 0
        print(f"resuming {s.name}: {s.n_clumps} clumps, vmax {np.linalg.norm(s.vel, axis=1).max():.4f}", flush=True)
        a.max_steps += steps
        if a.frictionless_sides:
            m0 = np.asarray(s.materials[0], float)
            s.materials = np.array([m0, [m0[0], m0[1], 0.0, m0[3]]])
            for pl in s.planes:
                if abs(pl.normal[2]) < 0.5:
                    pl.material = 1
            print("side walls frictionless (material 1: mu = 0)", flush=True)
    else:
        n = int(round(a.density * a.side * a.side * a.depth))
        vol = sum(c * t.mass / w.GRAIN_DENSITY for c, t in zip(w.ds_type_counts(n), w.ds_templates()))
        H = vol / a.fraction / (a.side * a.side)
        s = rsa_bed_exact(a.seed, n, (0.0, 0.0, 0.0), (a.side, a.side, H), vz=a.vz)
        print(f"spawned {n} clumps / {s.n_spheres} spheres in a {H:.3f} m column ({time.time() - t0:.1f}s)",
              flush=True)
        steps = 0
    o = oracle.Oracle(s, detect=1)
    while steps < a.max_steps:
        o.step(a.chunk)
        steps += a.chunk
        st = o.state()
        vmax = float(np.linalg.norm(st["vel"], axis=1).max())
        c = o.contacts()
        print(f"step {steps}: vmax {vmax:.4f} m/s, zmax {st['pos'][:, 2].max():.4f} m, "
              f"contacts {len(c['key_a'])} ({(c['delta'] > 0).sum()} touching), {time.time() - t0:.0f}s",
              flush=True)
        if steps % 20000 == 0 or (steps > 50000 and vmax < a.vstop) or steps >= a.max_steps:
            out = s.copy()
            out.pos, out.quat, out.vel, out.omega = st["pos"], st["quat"], st["vel"], st["omega"]
            out.domain_hi = np.array([a.side + 1e-3, a.side + 1e-3, st["pos"][:, 2].max() + 0.02])
            out.name = f"ds-patch-{int(a.side * 1e3)}mm-settled-{steps}"
            os.makedirs(os.path.dirname(os.path.abspath(a.out)), exist_ok=True)
            save_scene(a.out, out)
        if steps > 50000 and vmax < a.vstop:
            break
    print("done", steps, flush=True)


if __name__ == "__main__":
    main()
