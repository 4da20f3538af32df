"""Benchmark beds C4/C5: the oracle-settled DS patch copy-pasted to millions of clumps.

The patch (`data/ds_patch_30mm.npz`) is written by `workloads/make_patch.py`, which calls
only `oracle/`.  Tiles are laid out on an x-y lattice without gaps, each the mirror image of
its neighbours across their shared face (so the walls the patch settled against are replaced by
mirror images pressing back).  Extra clumps are trimmed from the top of the bed to hit the
target count exactly.  Nothing here computes forces or motion.
"""
from __future__ import annotations

import math
import os

import numpy as np

from .ds import C4_MATERIALS, M0, ds_templates
from .scenes import Scene, box_planes

HERE = os.path.dirname(os.path.abspath(__file__))
PATCH = os.path.join(HERE, "data", "ds_patch_30mm.npz")

C5_CLUMPS = 11_336_638  # P:574, VIPER-scale bed
C4_CLUMPS = 2_000_000


def _qmul(a, b):
    w1, x1, y1, z1 = a.T
    w2, x2, y2, z2 = b.T
    return np.stack([w1 * w2 - x1 * x2 - y1 * y2 - z1 * z2, w1 * x2 + x1 * w2 + y1 * z2 - z1 * y2,
                     w1 * y2 - x1 * z2 + y1 * w2 + z1 * x2, w1 * z2 + x1 * y2 - y1 * x2 + z1 * w2], axis=1)


def load_patch(path: str = PATCH) -> Scene:
    from .scenes import load_scene

    if not os.path.exists(path):
        raise FileNotFoundError(f"{path} missing: run `python -m workloads.make_patch` (oracle-only settling)")
    return load_scene(path)


def _mirror(pos, quat, vel, omega, axis, side):
    """The patch reflected across its mid-plane x = side/2 (axis 0) or y = side/2 (axis 1).  The DS
    templates are planar (body z offsets 0), so the mirror image of a clump is the same template
    with R' = M R D, D = diag(1, 1, -1) a proper rotation: q' = (M R M) then a half turn about the
    body axis M D; v' = M v; the angular velocity is a pseudo-vector, Omega_body' = -D Omega_body."""
    pos, quat, vel, omega = pos.copy(), quat.copy(), vel.copy(), omega.copy()
    pos[:, axis] = side - pos[:, axis]
    vel[:, axis] = -vel[:, axis]
    w, x, y, z = quat.T
    if axis == 0:  # M R M = q(w, x, -y, -z); M D = diag(-1, 1, -1) = half turn about body y
        q = np.stack([w, x, -y, -z], axis=1)
        half = np.array([[0.0, 0.0, 1.0, 0.0]])
    else:  # M R M = q(w, -x, y, -z); M D = diag(1, -1, -1) = half turn about body x
        q = np.stack([w, -x, y, -z], axis=1)
        half = np.array([[0.0, 1.0, 0.0, 0.0]])
    quat = _qmul(q, np.repeat(half, len(q), 0))
    omega[:, 0], omega[:, 1] = -omega[:, 0], -omega[:, 1]
    return pos, quat, vel, omega


def tiled_bed(n_target: int, footprint=(2.48, 1.0), seed: int = 574, per_comp_mat: bool = False,
              gap: float = 0.0, patch: Scene | None = None, vel_jitter: float = 0.0) -> Scene:
    """Tile the settled patch over `footprint` (rounded up to whole tiles) and trim to n_target clumps.

    Copy-paste of a settled patch.  Neighbouring tiles are mirror images of each other
    across their shared face (tile (i, j) is the patch reflected in x for odd i and in y for odd
    j), with no gap: a sphere the patch pressed against its side wall then meets its own mirror
    image, which pushes back along the wall normal like the wall did, so the tiles' force networks
    stay loaded.  (Plain translated copies with a gap left every tile a free-standing column whose
    lateral support was gone: the bed lost 90% of its contacts in its first 1000 steps.)"""
    p = load_patch() if patch is None else patch
    side_x = max(pl.point[0] for pl in p.planes if pl.normal[0] < 0)
    side_y = max(pl.point[1] for pl in p.planes if pl.normal[1] < 0)
    Lx, Ly = side_x + gap, side_y + gap
    nx = max(1, math.ceil(footprint[0] / Lx))
    ny = max(1, math.ceil(footprint[1] / Ly))
    while nx * ny * p.n_clumps < n_target:  # footprint too small for the count: widen along x
        nx += 1
    m = p.n_clumps
    T = nx * ny
    pos = np.empty((T, m, 3))
    quat = np.empty((T, m, 4))
    vel = np.empty((T, m, 3))
    om = np.empty((T, m, 3))
    ti, tj = np.divmod(np.arange(T), ny)
    for mx in (0, 1):
        for my in (0, 1):
            sel = np.nonzero(((ti & 1) == mx) & ((tj & 1) == my))[0]
            if sel.size == 0:
                continue
            P = (p.pos, p.quat, p.vel, p.omega)
            if mx:
                P = _mirror(*P, 0, side_x)
            if my:
                P = _mirror(*P, 1, side_y)
            pos[sel], quat[sel], vel[sel], om[sel] = P
    rng = np.random.default_rng(seed)
    pos[:, :, 0] += (ti * Lx)[:, None]
    pos[:, :, 1] += (tj * Ly)[:, None]
    pos = pos.reshape(-1, 3)
    quat = quat.reshape(-1, 4)
    vel = vel.reshape(-1, 3)
    om = om.reshape(-1, 3)
    tid = np.tile(p.tid, T).astype(np.int32)
    if n_target < pos.shape[0]:
        keep = np.sort(np.argsort(pos[:, 2], kind="stable")[:n_target])
        pos, quat, vel, om, tid = pos[keep], quat[keep], vel[keep], om[keep], tid[keep]
    if vel_jitter:
        vel = vel + rng.uniform(-vel_jitter, vel_jitter, size=vel.shape)
    quat /= np.linalg.norm(quat, axis=1, keepdims=True)
    n = pos.shape[0]
    lo = np.array([0.0, 0.0, 0.0])
    hi = np.array([nx * Lx - gap, ny * Ly - gap, float(pos[:, 2].max()) + 0.01])
    templates = ds_templates(per_component_materials=per_comp_mat)
    mats = np.array(C4_MATERIALS if per_comp_mat else [M0])
    return Scene(materials=mats, templates=templates, planes=box_planes(lo, hi, 0, top=False), h=p.h,
                 gravity=np.array([0.0, 0.0, -9.81]), domain_lo=lo - 1e-3, domain_hi=hi + np.array([1e-3, 1e-3, 0.05]),
                 gid=np.arange(n, dtype=np.int64), tid=tid, pos=pos, quat=quat, vel=vel, omega=om,
                 name=f"tiled-{nx}x{ny}-{n}")


def c5_bed(**kw) -> Scene:
    """Config 5: VIPER-scale bed, 11,336,638 DS clumps, footprint ~2.48 x 1.0 m, M0."""
    s = tiled_bed(C5_CLUMPS, footprint=(2.48, 1.0), **kw)
    s.name = "C5-viper-bed"
    return s


def c4_bed(**kw) -> Scene:
    """Config 4: GRC-1 DS bed, 2,000,000 clumps, footprint 0.66 x 0.66 m, per-sphere materials M_{k mod 4}."""
    s = tiled_bed(C4_CLUMPS, footprint=(0.66, 0.66), per_comp_mat=True, **kw)
    s.name = "C4-grc1-bed"
    return s


def crop(scene: Scene, lo, hi) -> Scene:
    """Clumps whose COM lies in the box [lo, hi] (a bounded sample of a bed)."""
    lo, hi = np.asarray(lo), np.asarray(hi)
    sel = np.nonzero(np.all((scene.pos >= lo) & (scene.pos <= hi), axis=1))[0]
    return scene.subset(sel)


def patch_mesh(cone_speed: float = 0.5, spin: float = 0.0, depth: float = 1.0e-3) -> Scene:
    """Mesh parity bed (NEXT-3): the settled 30 mm patch with its floor plane replaced by an 18-
    triangle mesh plate of another material, and a 24-facet 60-degree cone (base radius
    6 mm) whose apex starts `depth` below the bed surface, pushed down at `cone_speed` and
    optionally spun about its axis at `spin` rad/s."""
    from .scenes import MAT_B, Mesh, mesh_cone, mesh_rect

    s = load_patch()
    floor = [p for p in s.planes if p.normal[2] > 0.5][0]
    s.planes = [p for p in s.planes if not p.normal[2] > 0.5]
    for p in s.planes:  # the side walls in M0 (the patch settled against frictionless ones)
        p.material = 0
    s.materials = np.array([M0, MAT_B])
    side_x = max(pl.point[0] for pl in s.planes if pl.normal[0] < 0)
    side_y = max(pl.point[1] for pl in s.planes if pl.normal[1] < 0)
    cx, cy = 0.5 * side_x, 0.5 * side_y
    s.meshes = [Mesh(mesh_rect(side_x + 2e-3, side_y + 2e-3, 3, 3), 1, pos=(cx, cy, float(floor.point[2])))]
    rc = 6e-3
    hc = rc / math.tan(math.radians(30.0))
    near = np.hypot(s.pos[:, 0] - cx, s.pos[:, 1] - cy) < 5e-3
    top = float(s.pos[near, 2].max())
    s.meshes.append(Mesh(mesh_cone(rc, hc, 24), 0, pos=(cx + 0.37e-3, cy - 0.21e-3, top - depth),
                         vel=(0.0, 0.0, -cone_speed), omega=(0.0, 0.0, spin)))
    s.domain_hi = np.array(s.domain_hi, dtype=float) + np.array([0.0, 0.0, hc + 0.02])
    s.name = "patch-mesh"
    return s


def c3_impact(seed: int = 33) -> Scene:
    """Config 3 at impact (a parity case, not a bench line): the C3 column (100k DS clumps, RSA
    in the r = 6 cm cylinder) lowered onto a settled base layer — the oracle-settled patch tiled
    under the column and cut to the same cylinder, as the first arrivals of the pour would have
    built it — every column clump falling at 2 m/s (a 20 cm drop) with +-2 m/s of random relative
    motion and +-200 rad/s of random spin.  Its lowest sphere starts 2 um into the top of the
    base layer, so high-speed impacts on a dense layer begin at once while the sparse column
    above keeps falling."""
    from scipy.spatial.transform import Rotation

    from .scenes import c3_repose

    col = c3_repose()
    rng = np.random.default_rng(seed)
    base = tiled_bed(60_000, footprint=(0.125, 0.125), seed=seed)
    c = 0.5 * (base.domain_lo[:2] + base.domain_hi[:2])
    keep = np.nonzero(np.hypot(base.pos[:, 0] - c[0], base.pos[:, 1] - c[1]) < 0.06)[0]
    base = base.subset(keep)
    base.pos = base.pos - np.array([c[0], c[1], 0.0])

    def sphere_extent(s, sel, lowest):
        R = Rotation.from_quat(s.quat[sel][:, [1, 2, 3, 0]]).as_matrix()
        z = [float(s.pos[i, 2] + (R[k] @ o)[2] + (-r if lowest else r)) for k, i in enumerate(sel)
             for o, r in zip(s.templates[s.tid[i]].offsets, s.templates[s.tid[i]].radius)]
        return min(z) if lowest else max(z)

    top = sphere_extent(base, np.argsort(base.pos[:, 2])[-500:], False)
    bottom = sphere_extent(col, np.argsort(col.pos[:, 2])[:500], True)
    col.pos = col.pos + np.array([0.0, 0.0, top - bottom - 2e-6])
    n0 = base.n_clumps
    vel = np.concatenate([base.vel, np.column_stack([np.zeros(col.n_clumps), np.zeros(col.n_clumps),
                                                     np.full(col.n_clumps, -2.0)])
                          + rng.uniform(-2.0, 2.0, size=(col.n_clumps, 3))])
    om = np.concatenate([base.omega, rng.uniform(-200.0, 200.0, size=(col.n_clumps, 3))])
    s = col.copy()
    s.gid = np.concatenate([np.arange(n0, dtype=np.int64), col.gid + n0])
    s.tid = np.concatenate([base.tid, col.tid]).astype(np.int32)
    s.pos = np.concatenate([base.pos, col.pos])
    s.quat = np.concatenate([base.quat, col.quat])
    s.vel, s.omega = vel, om
    s.domain_hi = np.array([s.domain_hi[0], s.domain_hi[1], float(col.pos[:, 2].max()) + 0.05])
    s.name = "C3-impact"
    return s
