"""Seeded synthetic scenes (the configs of BASELINE.json) — inputs only, no method arithmetic.

Every scene is a `Scene`: material table, clump templates (with mass/inertia),
fixed planes, solver parameters and the initial clump state.  The same Scene is
handed unchanged to the CPU oracle (`oracle/`) and to the CUDA library
(`paper_2307_03445_b200`); neither side imports the other.

Input recipe (DESIGN.md §"Input recipe"):
* C1  `c1_box`: 1,000 DS type-7 clumps on a 10x10x10 jittered lattice (pitch 2.6 mm,
  jitter +-0.02 mm), uniform random orientation (Shoemake), V ~ U(-0.5,0.5) m/s,
  Omega = 0, six walls 0.05 mm outside the lattice's bounding spheres, material M0,
  gravity (0,0,-9.81), h = 1e-6 s.
* C2  `c2_head_on` / `c2_wall`: two single-sphere clumps (r = 1 mm, rho = 2600)
  head-on along x, or one sphere falling normally onto a plane, g = 0.
* random scenes for contact-set checks: polydisperse spheres / DS clumps in a box.
* beds: random sequential addition (RSA) of DS bounding spheres in a box with the
  Table-1 number fractions; a settled patch (written by `workloads/make_patch.py`,
  which only calls `oracle/`) tiled by copy-paste for C4/C5.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field, replace

import numpy as np

from .ds import (C4_MATERIALS, DS_NCOMP, M0, Template, ds_number_fractions, ds_template,
                 ds_templates, ds_type_counts, sphere_template)

INT64_MAX = np.iinfo(np.int64).max
GID_STRIDE = 64  # sphere gid = clump_gid * 64 + component


@dataclass
class Mesh:
    """A kinematic triangle mesh (NEXT-3): triangles in the body frame, prescribed motion."""
    verts: np.ndarray  # (n_tri, 3, 3) body-frame vertices (a, b, c)
    material: int = 0
    pos: tuple = (0.0, 0.0, 0.0)  # reference point X (world)
    quat: tuple = (1.0, 0.0, 0.0, 0.0)  # body -> world
    vel: tuple = (0.0, 0.0, 0.0)  # world
    omega: tuple = (0.0, 0.0, 0.0)  # world, about X


@dataclass
class Plane:
    point: tuple
    normal: tuple  # unit, pointing into the domain
    material: int = 0


@dataclass
class Scene:
    materials: np.ndarray  # (n_mat, 4): E, nu, mu, CoR
    templates: list
    planes: list
    h: float
    gravity: np.ndarray
    domain_lo: np.ndarray
    domain_hi: np.ndarray
    margin: float = 0.0
    cell_size: float = 0.0  # 0 = library chooses
    # state
    gid: np.ndarray = None  # (n,) int64 clump gids
    tid: np.ndarray = None  # (n,) int32 template ids
    pos: np.ndarray = None  # (n,3)
    quat: np.ndarray = None  # (n,4) (w,x,y,z), Hamilton, body->world
    vel: np.ndarray = None  # (n,3) world
    omega: np.ndarray = None  # (n,3) body frame
    name: str = ""
    meshes: list = field(default_factory=list)  # kinematic triangle meshes (NEXT-3)

    @property
    def n_clumps(self) -> int:
        return int(self.gid.shape[0])

    @property
    def n_spheres(self) -> int:
        nc = np.array([t.n_comp for t in self.templates])
        return int(nc[self.tid].sum()) if self.n_clumps else 0

    def template_arrays(self):
        """Flattened template table: n_comp, offsets(3*total), radius, material, mass, inertia(3*nt)."""
        ncomp = np.array([t.n_comp for t in self.templates], dtype=np.int32)
        offs = np.concatenate([t.offsets.reshape(-1) for t in self.templates]).astype(np.float64)
        rad = np.concatenate([t.radius for t in self.templates]).astype(np.float64)
        mat = np.concatenate([t.material for t in self.templates]).astype(np.int32)
        mass = np.array([t.mass for t in self.templates], dtype=np.float64)
        inertia = np.concatenate([t.inertia for t in self.templates]).astype(np.float64)
        return ncomp, offs, rad, mat, mass, inertia

    def plane_arrays(self):
        if not self.planes:
            return (np.zeros((0, 3)), np.zeros((0, 3)), np.zeros(0, dtype=np.int32))
        pts = np.array([p.point for p in self.planes], dtype=np.float64)
        nrm = np.array([p.normal for p in self.planes], dtype=np.float64)
        mat = np.array([p.material for p in self.planes], dtype=np.int32)
        return pts, nrm, mat

    def copy(self) -> "Scene":
        return replace(self, gid=self.gid.copy(), tid=self.tid.copy(), pos=self.pos.copy(),
                       quat=self.quat.copy(), vel=self.vel.copy(), omega=self.omega.copy(),
                       planes=list(self.planes), templates=list(self.templates), meshes=list(self.meshes))

    def subset(self, idx) -> "Scene":
        s = self.copy()
        s.gid, s.tid, s.pos = self.gid[idx].copy(), self.tid[idx].copy(), self.pos[idx].copy()
        s.quat, s.vel, s.omega = self.quat[idx].copy(), self.vel[idx].copy(), self.omega[idx].copy()
        return s


# ------------------------------------------------------------------ helpers
def random_quaternions(rng: np.random.Generator, n: int) -> np.ndarray:
    """Uniform random unit quaternions (Shoemake), returned as (w,x,y,z)."""
    u1, u2, u3 = rng.random(n), rng.random(n), rng.random(n)
    a, b = np.sqrt(1.0 - u1), np.sqrt(u1)
    q = np.stack([b * np.cos(2 * np.pi * u3), a * np.sin(2 * np.pi * u2),
                  a * np.cos(2 * np.pi * u2), b * np.sin(2 * np.pi * u3)], axis=1)
    return q / np.linalg.norm(q, axis=1, keepdims=True)


def box_planes(lo, hi, material: int = 0, top: bool = True) -> list:
    """Axis-aligned box walls with inward normals (floor first)."""
    lo, hi = np.asarray(lo, float), np.asarray(hi, float)
    pl = [Plane((0.0, 0.0, lo[2]), (0.0, 0.0, 1.0), material),
          Plane((lo[0], 0.0, 0.0), (1.0, 0.0, 0.0), material),
          Plane((hi[0], 0.0, 0.0), (-1.0, 0.0, 0.0), material),
          Plane((0.0, lo[1], 0.0), (0.0, 1.0, 0.0), material),
          Plane((0.0, hi[1], 0.0), (0.0, -1.0, 0.0), material)]
    if top:
        pl.append(Plane((0.0, 0.0, hi[2]), (0.0, 0.0, -1.0), material))
    return pl


def _mk_state(n):
    return (np.arange(n, dtype=np.int64), np.zeros(n, np.int32), np.zeros((n, 3)),
            np.tile(np.array([1.0, 0.0, 0.0, 0.0]), (n, 1)), np.zeros((n, 3)), np.zeros((n, 3)))


# ------------------------------------------------------------------ C1
def c1_box(seed: int = 1, n_side: int = 10, pitch: float = 2.6e-3, jitter: float = 0.02e-3,
           vmax: float = 0.5, h: float = 1e-6) -> Scene:
    """Config 1: 1,000 three-sphere (DS type 7) clumps settling in a box."""
    rng = np.random.default_rng(seed)
    t7 = ds_template(6, 0)
    n = n_side ** 3
    g = np.arange(n_side) * pitch
    P = np.stack(np.meshgrid(g, g, g, indexing="ij"), axis=-1).reshape(-1, 3)
    P = P + rng.uniform(-jitter, jitter, size=P.shape)
    gid, tid, pos, quat, vel, om = _mk_state(n)
    pos[:] = P
    quat[:] = random_quaternions(rng, n)
    vel[:] = rng.uniform(-vmax, vmax, size=(n, 3))
    rb = t7.bounding_radius
    lo = np.full(3, -rb - 0.05e-3)
    hi = np.full(3, (n_side - 1) * pitch + rb + 0.05e-3)
    dom_pad = 2e-3
    return Scene(materials=np.array([M0]), templates=[t7], planes=box_planes(lo, hi), h=h,
                 gravity=np.array([0.0, 0.0, -9.81]), domain_lo=lo - dom_pad, domain_hi=hi + dom_pad,
                 gid=gid, tid=tid, pos=pos, quat=quat, vel=vel, omega=om, name="C1")


# ------------------------------------------------------------------ C2
MAT_A = (1.0e9, 0.3, 0.4, 0.5)
MAT_B = (2.0e9, 0.25, 0.3, 0.8)


def c2_head_on(v0: float = 1.0, mat_a=MAT_A, mat_b=MAT_B, mats=(0, 0), radius: float = 1e-3,
               h: float = 1e-6, gap: float = 0.0) -> Scene:
    """Config 2(i): two single-sphere clumps head-on along x, relative speed v0, g = 0.

    Sphere 0 at -(r + gap/2) moving +v0/2, sphere 1 at +(r + gap/2) moving -v0/2.
    """
    ta = sphere_template(radius, mats[0])
    tb = sphere_template(radius, mats[1])
    gid, tid, pos, quat, vel, om = _mk_state(2)
    tid[:] = [0, 1]
    pos[0] = (-(radius + gap / 2), 0.0, 0.0)
    pos[1] = (radius + gap / 2, 0.0, 0.0)
    vel[0] = (v0 / 2, 0.0, 0.0)
    vel[1] = (-v0 / 2, 0.0, 0.0)
    L = 10 * radius
    return Scene(materials=np.array([mat_a, mat_b]), templates=[ta, tb], planes=[], h=h,
                 gravity=np.zeros(3), domain_lo=np.full(3, -L), domain_hi=np.full(3, L),
                 gid=gid, tid=tid, pos=pos, quat=quat, vel=vel, omega=om, name="C2-head-on")


def c2_wall(v0: float = 1.0, mat_sphere=MAT_A, mat_wall=MAT_B, radius: float = 1e-3, h: float = 1e-6,
            gap: float = 0.0) -> Scene:
    """Config 2(ii): one sphere (material 0) moving at -v0 along z onto the plane z=0 (material 1)."""
    t = sphere_template(radius, 0)
    gid, tid, pos, quat, vel, om = _mk_state(1)
    pos[0] = (0.0, 0.0, radius + gap)
    vel[0] = (0.0, 0.0, -v0)
    L = 10 * radius
    return Scene(materials=np.array([mat_sphere, mat_wall]), templates=[t],
                 planes=[Plane((0.0, 0.0, 0.0), (0.0, 0.0, 1.0), 1)], h=h, gravity=np.zeros(3),
                 domain_lo=np.array([-L, -L, -L]), domain_hi=np.full(3, L),
                 gid=gid, tid=tid, pos=pos, quat=quat, vel=vel, omega=om, name="C2-wall")


# ------------------------------------------------------------------ random scenes
def random_spheres(seed: int, n: int, box: float = 0.02, rmin: float = 0.7e-3, rmax: float = 3.6e-3,
                   vmax: float = 0.5, n_mat: int = 1, walls: bool = True, h: float = 1e-6) -> Scene:
    """n single-sphere clumps with random radii (up to 8 distinct sizes), positions, velocities."""
    rng = np.random.default_rng(seed)
    sizes = np.unique(np.round(rng.uniform(rmin, rmax, size=min(8, n)), 6))
    templates = [sphere_template(float(r), int(i % n_mat)) for i, r in enumerate(sizes)]
    gid, tid, pos, quat, vel, om = _mk_state(n)
    gid[:] = rng.permutation(n).astype(np.int64) * 3 + 5  # non-contiguous gids
    tid[:] = rng.integers(0, len(templates), n)
    pos[:] = rng.uniform(0.0, box, size=(n, 3))
    quat[:] = random_quaternions(rng, n)
    vel[:] = rng.uniform(-vmax, vmax, size=(n, 3))
    om[:] = rng.uniform(-50, 50, size=(n, 3))
    mats = [M0, (5.0e8, 0.25, 0.3, 0.6), (2.0e9, 0.35, 0.5, 0.4), (1.0e9, 0.3, 0.6, 0.7)][:n_mat]
    planes = box_planes(np.zeros(3), np.full(3, box), 0) if walls else []
    pad = 5e-3
    return Scene(materials=np.array(mats), templates=templates, planes=planes, h=h,
                 gravity=np.array([0.0, 0.0, -9.81]), domain_lo=np.full(3, -pad),
                 domain_hi=np.full(3, box + pad), gid=gid, tid=tid, pos=pos, quat=quat, vel=vel,
                 omega=om, name=f"random-spheres-{n}")


def random_clumps(seed: int, n: int, box: float = 0.03, vmax: float = 0.5, per_comp_mat: bool = True,
                  walls: bool = True, h: float = 1e-6, types=None) -> Scene:
    """n DS clumps (types drawn by number fraction) at random poses; overlaps allowed."""
    rng = np.random.default_rng(seed)
    templates = ds_templates(per_component_materials=per_comp_mat)
    gid, tid, pos, quat, vel, om = _mk_state(n)
    gid[:] = rng.permutation(n).astype(np.int64) + 1000
    if types is None:
        tid[:] = rng.choice(7, size=n, p=ds_number_fractions())
    else:
        tid[:] = rng.choice(np.asarray(types), size=n)
    pos[:] = rng.uniform(0.0, box, size=(n, 3))
    quat[:] = random_quaternions(rng, n)
    vel[:] = rng.uniform(-vmax, vmax, size=(n, 3))
    om[:] = rng.uniform(-100, 100, size=(n, 3))
    mats = C4_MATERIALS if per_comp_mat else [M0]
    planes = box_planes(np.zeros(3), np.full(3, box), 0) if walls else []
    pad = 15e-3
    return Scene(materials=np.array(mats), templates=templates, planes=planes, h=h,
                 gravity=np.array([0.0, 0.0, -9.81]), domain_lo=np.full(3, -pad),
                 domain_hi=np.full(3, box + pad), gid=gid, tid=tid, pos=pos, quat=quat, vel=vel,
                 omega=om, name=f"random-clumps-{n}")


# ------------------------------------------------------------------ RSA beds
def rsa_bed(seed: int, n_clumps: int, lo, hi, per_comp_mat: bool = False, vz: float = 0.0,
            h: float = 1e-6, top_wall: bool = False, cylinder_r: float = 0.0,
            domain_pad=(0.0, 0.0, 0.0), max_tries: int = 200) -> Scene:
    """Random sequential addition of DS clump bounding spheres inside [lo, hi] (largest first).

    Non-overlapping bounding spheres, random orientations; Table-1 number fractions
    (fact 0.1-5).  If `cylinder_r` > 0 the centres are restricted to a vertical
    cylinder about the box's x-y centre (C3 repose column).
    """
    from scipy.spatial import cKDTree

    rng = np.random.default_rng(seed)
    templates = ds_templates(per_component_materials=per_comp_mat)
    rb = np.array([t.bounding_radius for t in templates])
    counts = ds_type_counts(n_clumps)
    types = np.concatenate([np.full(c, t, dtype=np.int32) for t, c in enumerate(counts)])
    lo, hi = np.asarray(lo, float), np.asarray(hi, float)
    cx, cy = 0.5 * (lo[0] + hi[0]), 0.5 * (lo[1] + hi[1])
    # batched RSA, one radius at a time (largest first): propose a batch of centres, drop those
    # that overlap a placed sphere (k-d tree query) or an earlier accepted proposal of the same
    # batch, keep what is needed; a seeded, valid non-overlapping packing
    P = np.zeros((0, 3))
    Rp = np.zeros(0)
    for t in np.argsort(-rb, kind="stable"):
        r, need = rb[t], int(counts[t])
        fails = 0
        while need > 0:
            m = int(min(max(4 * need, 2048), 400_000))
            q = rng.uniform(lo + r, hi - r, size=(m, 3))
            if cylinder_r > 0:
                q = q[(q[:, 0] - cx) ** 2 + (q[:, 1] - cy) ** 2 <= (cylinder_r - r) ** 2]
            if P.shape[0]:
                tree = cKDTree(P)
                near = tree.query_ball_point(q, r + Rp.max(), workers=-1)
                ok = np.ones(q.shape[0], bool)
                for i, js in enumerate(near):
                    if js:
                        js = np.asarray(js)
                        if np.any(np.sum((P[js] - q[i]) ** 2, axis=1) < (Rp[js] + r) ** 2):
                            ok[i] = False
                q = q[ok]
            if q.shape[0]:
                clash = cKDTree(q).query_pairs(2 * r, output_type="ndarray")
                keep = np.ones(q.shape[0], bool)
                if clash.size:
                    bad_with = {}
                    for a, b in clash:
                        bad_with.setdefault(int(max(a, b)), []).append(int(min(a, b)))
                    for i in sorted(bad_with):
                        if any(keep[j] for j in bad_with[i]):
                            keep[i] = False
                q = q[keep][:need]
            if q.shape[0] == 0:
                fails += 1
                if fails > max_tries // 100 + 3:
                    raise RuntimeError(f"RSA could not place {need} clumps of type {t}; box too small")
                continue
            P = np.concatenate([P, q])
            Rp = np.concatenate([Rp, np.full(q.shape[0], r)])
            need -= q.shape[0]
    types = np.repeat(np.argsort(-rb, kind="stable"), counts[np.argsort(-rb, kind="stable")]).astype(np.int32)
    gid, tid, pos, quat, vel, om = _mk_state(n_clumps)
    perm = rng.permutation(n_clumps)
    tid[:] = types[perm]
    pos[:] = P[perm]
    quat[:] = random_quaternions(rng, n_clumps)
    vel[:, 2] = vz
    mats = C4_MATERIALS if per_comp_mat else [M0]
    dom_lo = lo - np.asarray(domain_pad)
    dom_hi = hi + np.asarray(domain_pad)
    return Scene(materials=np.array(mats), templates=templates,
                 planes=box_planes(lo, hi, 0, top=top_wall), h=h, gravity=np.array([0.0, 0.0, -9.81]),
                 domain_lo=dom_lo, domain_hi=dom_hi, gid=gid, tid=tid, pos=pos, quat=quat, vel=vel,
                 omega=om, name=f"rsa-bed-{n_clumps}")


def rsa_bed_exact(seed: int, n_clumps: int, lo, hi, per_comp_mat: bool = False, vz: float = 0.0,
                  h: float = 1e-6, clearance: float = 0.05e-3, max_tries: int = 5000) -> Scene:
    """RSA with the clumps' actual component spheres (not bounding spheres): denser spawn.

    Clumps are placed largest type first at uniform random poses inside [lo, hi]; a pose
    is accepted when every component sphere clears every placed sphere by `clearance`
    and stays inside the box.  Sphere centres for the test use scipy's Rotation, so
    this module still holds none of the method's own arithmetic.
    """
    from scipy.spatial.transform import Rotation

    rng = np.random.default_rng(seed)
    templates = ds_templates(per_component_materials=per_comp_mat)
    counts = ds_type_counts(n_clumps)
    types = np.concatenate([np.full(c, t, dtype=np.int32) for t, c in enumerate(counts)])
    lo, hi = np.asarray(lo, float), np.asarray(hi, float)
    n_sph = int(sum(templates[t].n_comp for t in types))
    S = np.full((n_sph, 3), 1e9)
    Sr = np.zeros(n_sph)
    ns = 0
    P = np.zeros((n_clumps, 3))
    Q = np.zeros((n_clumps, 4))
    for k, t in enumerate(types):
        tpl = templates[t]
        rb = tpl.bounding_radius
        ok = False
        for _ in range(max_tries):
            p = rng.uniform(lo + rb * np.array([0.3, 0.3, 0.3]), hi - rb * np.array([0.3, 0.3, 0.3]))
            q = random_quaternions(rng, 1)[0]
            c = p + Rotation.from_quat(q[[1, 2, 3, 0]]).apply(tpl.offsets)
            r = tpl.radius
            if np.any(c - r[:, None] < lo + clearance) or np.any(c + r[:, None] > hi - clearance):
                continue
            if ns:
                near = np.all(np.abs(S[:ns] - p) < rb + 3.7e-3 + clearance, axis=1)
                if near.any():
                    d = np.linalg.norm(S[:ns][near][None, :, :] - c[:, None, :], axis=-1)
                    if np.any(d < r[:, None] + Sr[:ns][near][None, :] + clearance):
                        continue
            ok = True
            break
        if not ok:
            raise RuntimeError(f"RSA could not place clump {k} of {n_clumps}")
        S[ns:ns + tpl.n_comp] = c
        Sr[ns:ns + tpl.n_comp] = tpl.radius
        ns += tpl.n_comp
        P[k], Q[k] = p, q
    gid, tid, pos, quat, vel, om = _mk_state(n_clumps)
    perm = rng.permutation(n_clumps)
    tid[:] = types[perm]
    pos[:] = P[perm]
    quat[:] = Q[perm]
    vel[:, 2] = vz
    mats = C4_MATERIALS if per_comp_mat else [M0]
    return Scene(materials=np.array(mats), templates=templates, planes=box_planes(lo, hi, 0, top=False), h=h,
                 gravity=np.array([0.0, 0.0, -9.81]), domain_lo=lo - 1e-3, domain_hi=hi + np.array([1e-3, 1e-3, 0.05]),
                 gid=gid, tid=tid, pos=pos, quat=quat, vel=vel, omega=om, name=f"rsa-exact-{n_clumps}")


def c3_repose(seed: int = 3, n_clumps: int = 100_000, h: float = 1e-6) -> Scene:
    """Config 3: 100k DS clumps in a vertical cylinder r = 0.06 m above the plane z = 0,
    solid fraction of bounding spheres ~0.25 (column ~0.57 m); far walls at +-0.3 m."""
    templates = ds_templates()
    rb = np.array([t.bounding_radius for t in templates])
    vol = float(np.sum(ds_type_counts(n_clumps) * 4.0 / 3.0 * np.pi * rb ** 3))
    height = vol / 0.25 / (np.pi * 0.06 ** 2)
    s = rsa_bed(seed, n_clumps, lo=(-0.06, -0.06, 0.005), hi=(0.06, 0.06, 0.005 + height),
                cylinder_r=0.06, h=h, max_tries=2000)
    s.planes = [Plane((0.0, 0.0, 0.0), (0.0, 0.0, 1.0), 0),
                Plane((-0.3, 0.0, 0.0), (1.0, 0.0, 0.0), 0), Plane((0.3, 0.0, 0.0), (-1.0, 0.0, 0.0), 0),
                Plane((0.0, -0.3, 0.0), (0.0, 1.0, 0.0), 0), Plane((0.0, 0.3, 0.0), (0.0, -1.0, 0.0), 0)]
    s.domain_lo = np.array([-0.31, -0.31, -0.01])
    s.domain_hi = np.array([0.31, 0.31, 0.02 + height])
    s.name = "C3"
    return s


# ------------------------------------------------------------------ tiling (P:233 copy-paste)
def tile_scene(patch: Scene, nx: int, ny: int, gap: float = 0.2e-3, n_target: int | None = None,
               per_comp_mat: bool | None = None, walls_top: bool = False) -> Scene:
    """Copy-paste `patch` (whose clumps lie in its domain footprint) nx x ny times in x-y.

    Tiles are offset by (patch footprint + gap); gids are renumbered tile-major.
    If `n_target` is given, clumps are dropped from the last tiles' top to hit it.
    """
    pl = patch.planes
    lo = np.array([min(p.point[0] for p in pl if p.normal[0] > 0), min(p.point[1] for p in pl if p.normal[1] > 0),
                   min(p.point[2] for p in pl if p.normal[2] > 0)])
    hi = np.array([max(p.point[0] for p in pl if p.normal[0] < 0), max(p.point[1] for p in pl if p.normal[1] < 0)])
    Lx, Ly = hi[0] - lo[0] + gap, hi[1] - lo[1] + gap
    n = patch.n_clumps
    reps = []
    for i in range(nx):
        for j in range(ny):
            reps.append((i * Lx, j * Ly))
    off = np.array(reps)
    pos = (patch.pos[None, :, :] + np.concatenate([off, np.zeros((len(reps), 1))], axis=1)[:, None, :]).reshape(-1, 3)
    N = pos.shape[0]
    tid = np.tile(patch.tid, len(reps))
    quat = np.tile(patch.quat, (len(reps), 1))
    vel = np.tile(patch.vel, (len(reps), 1))
    om = np.tile(patch.omega, (len(reps), 1))
    if n_target is not None and n_target < N:
        # keep a deterministic subset: drop the highest clumps of the whole bed
        keep = np.sort(np.argsort(pos[:, 2], kind="stable")[:n_target])
        pos, tid, quat, vel, om = pos[keep], tid[keep], quat[keep], vel[keep], om[keep]
        N = n_target
    gid = np.arange(N, dtype=np.int64)
    blo = np.array([lo[0], lo[1], lo[2]])
    bhi = np.array([lo[0] + nx * Lx - gap, lo[1] + ny * Ly - gap, pos[:, 2].max() + 0.02])
    templates = patch.templates
    materials = patch.materials
    if per_comp_mat is not None:
        templates = ds_templates(per_component_materials=per_comp_mat)
        materials = np.array(C4_MATERIALS if per_comp_mat else [M0])
    return Scene(materials=materials, templates=templates, planes=box_planes(blo, bhi, 0, top=walls_top),
                 h=patch.h, gravity=patch.gravity.copy(), domain_lo=blo - np.array([1e-3, 1e-3, 1e-3]),
                 domain_hi=bhi + np.array([1e-3, 1e-3, 0.05]), gid=gid, tid=tid.astype(np.int32), pos=pos,
                 quat=quat, vel=vel, omega=om, name=f"tiled-{nx}x{ny}")


def save_scene(path: str, s: Scene) -> None:
    ncomp, offs, rad, mat, mass, inertia = s.template_arrays()
    pts, nrm, pmat = s.plane_arrays()
    np.savez_compressed(path, materials=s.materials, ncomp=ncomp, offs=offs, rad=rad, mat=mat, mass=mass,
                        inertia=inertia, plane_pts=pts, plane_nrm=nrm, plane_mat=pmat, h=s.h,
                        gravity=s.gravity, domain_lo=s.domain_lo, domain_hi=s.domain_hi, margin=s.margin,
                        cell_size=s.cell_size, gid=s.gid, tid=s.tid, pos=s.pos, quat=s.quat, vel=s.vel,
                        omega=s.omega, name=s.name)


def load_scene(path: str) -> Scene:
    z = np.load(path, allow_pickle=False)
    ncomp = z["ncomp"]
    templates = []
    o = 0
    for t, n in enumerate(ncomp):
        templates.append(Template(offsets=z["offs"][3 * o:3 * (o + n)].reshape(n, 3).copy(),
                                  radius=z["rad"][o:o + n].copy(), material=z["mat"][o:o + n].copy(),
                                  mass=float(z["mass"][t]), inertia=z["inertia"][3 * t:3 * t + 3].copy()))
        o += n
    planes = [Plane(tuple(p), tuple(nn), int(m)) for p, nn, m in zip(z["plane_pts"], z["plane_nrm"], z["plane_mat"])]
    return Scene(materials=z["materials"], templates=templates, planes=planes, h=float(z["h"]),
                 gravity=z["gravity"], domain_lo=z["domain_lo"], domain_hi=z["domain_hi"],
                 margin=float(z["margin"]), cell_size=float(z["cell_size"]), gid=z["gid"], tid=z["tid"],
                 pos=z["pos"], quat=z["quat"], vel=z["vel"], omega=z["omega"], name=str(z["name"]))


# ------------------------------------------------------------------ triangle meshes (NEXT-3)
def mesh_rect(lx: float, ly: float, nx: int = 1, ny: int = 1) -> np.ndarray:
    """A flat rectangle [-lx/2, lx/2] x [-ly/2, ly/2] in the body x-y plane, normal +z (counter-
    clockwise from above), split into nx x ny cells of two triangles each."""
    xs, ys = np.linspace(-lx / 2, lx / 2, nx + 1), np.linspace(-ly / 2, ly / 2, ny + 1)
    tris = []
    for i in range(nx):
        for j in range(ny):
            a, b = (xs[i], ys[j], 0.0), (xs[i + 1], ys[j], 0.0)
            c, d = (xs[i + 1], ys[j + 1], 0.0), (xs[i], ys[j + 1], 0.0)
            tris += [(a, b, c), (a, c, d)]
    return np.array(tris, dtype=np.float64)


def mesh_cone(radius: float, height: float, n: int = 24) -> np.ndarray:
    """The lateral surface of a cone with its apex at the body origin pointing down (-z) and a
    base circle of `radius` at z = height (the penetrometer tip of P:277: 60 deg opening for
    radius = height tan 30 deg), n facets, outward normals."""
    th = np.linspace(0.0, 2 * np.pi, n + 1)
    tris = []
    for k in range(n):
        p0 = (radius * np.cos(th[k]), radius * np.sin(th[k]), height)
        p1 = (radius * np.cos(th[k + 1]), radius * np.sin(th[k + 1]), height)
        tris.append(((0.0, 0.0, 0.0), p1, p0))
    return np.array(tris, dtype=np.float64)


def sphere_on_mesh(material_sphere=0, material_mesh=0, r: float = 1e-3, drop: float = 0.0, v0=(0.0, 0.0, 0.0),
                   mesh_vel=(0.0, 0.0, 0.0), mesh_omega=(0.0, 0.0, 0.0), g=(0.0, 0.0, -9.81), h: float = 1e-6,
                   with_plane: bool = False, materials=None, at=(0.3e-3, -0.2e-3)) -> Scene:
    """One sphere clump (rho 2600) above a 10 x 10 mm mesh square at z = 0 (or, with_plane,
    above the analytic plane z = 0 instead): gap `drop`, velocity v0."""
    mats = np.array(materials if materials is not None else [M0])
    t = sphere_template(r, material_sphere)
    gid, tid, pos, quat, vel, om = _mk_state(1)
    pos[0] = (at[0], at[1], r + drop)
    vel[0] = v0
    s = Scene(materials=mats, templates=[t], planes=[], h=h, gravity=np.array(g, float),
              domain_lo=np.array([-0.02, -0.02, -0.01]), domain_hi=np.array([0.02, 0.02, 0.03]), gid=gid, tid=tid,
              pos=pos, quat=quat, vel=vel, omega=om, name="sphere-on-mesh")
    if with_plane:
        s.planes = [Plane((0.0, 0.0, 0.0), (0.0, 0.0, 1.0), material_mesh)]
    else:
        s.meshes = [Mesh(mesh_rect(0.01, 0.01, 2, 2), material_mesh, vel=tuple(mesh_vel), omega=tuple(mesh_omega))]
    return s


def c1_mesh(seed: int = 1, cone_speed: float = 1.0, spin: float = 0.0) -> Scene:
    """The C1 box with two kinematic meshes (NEXT-3): its floor replaced by a 3 x 3-cell mesh plate
    (18 triangles, a different material) and a 24-facet 60-degree cone (the P:277 penetrometer
    tip: base radius 4 mm, apex down) entering the top layer at `cone_speed`, optionally spinning
    about its axis at `spin` rad/s (a wheel-like moving boundary)."""
    s = c1_box(seed)
    lo = np.array([p.point[2] for p in s.planes if p.normal[2] > 0.5])[0]
    s.planes = [p for p in s.planes if not p.normal[2] > 0.5]
    s.materials = np.array([M0, MAT_B])
    side = float(s.domain_hi[0] - s.domain_lo[0])
    c = 0.5 * (s.domain_lo + s.domain_hi)
    s.meshes.append(Mesh(mesh_rect(side, side, 3, 3), 1, pos=(float(c[0]), float(c[1]), float(lo))))
    top = float(s.pos[:, 2].max())
    rc = 4e-3
    hc = rc / math.tan(math.radians(30.0))
    s.meshes.append(Mesh(mesh_cone(rc, hc, 24), 0, pos=(float(c[0]) + 0.4e-3, float(c[1]) - 0.3e-3, top - 0.5e-3),
                         vel=(0.0, 0.0, -cone_speed), omega=(0.0, 0.0, spin)))
    s.domain_hi = s.domain_hi + np.array([0.0, 0.0, hc + 2e-3])
    s.name = "C1-mesh"
    return s


def mesh_funnel(r_top: float, r_bottom: float, height: float, n: int = 32) -> np.ndarray:
    """A conical hopper (frustum side wall, open at both ends): radius r_bottom at body z = 0 and
    r_top at z = height, n facets of two triangles."""
    th = np.linspace(0.0, 2 * np.pi, n + 1)
    tris = []
    for k in range(n):
        a = (r_bottom * np.cos(th[k]), r_bottom * np.sin(th[k]), 0.0)
        b = (r_bottom * np.cos(th[k + 1]), r_bottom * np.sin(th[k + 1]), 0.0)
        c = (r_top * np.cos(th[k + 1]), r_top * np.sin(th[k + 1]), height)
        d = (r_top * np.cos(th[k]), r_top * np.sin(th[k]), height)
        tris += [(a, b, c), (a, c, d)]
    return np.array(tris, dtype=np.float64)


def mesh_wheel(radius: float = 0.25, width: float = 0.15, n: int = 72, grousers: int = 24,
               grouser_h: float = 0.01) -> np.ndarray:
    """A rover-style wheel: the rolling surface of a cylinder about the body y axis
    (n facets around), its two side disks, and `grousers` radial plates of height grouser_h
    across the width.  Outward orientation is not needed (contacts are unsigned)."""
    th = np.linspace(0.0, 2 * np.pi, n + 1)
    y0, y1 = -0.5 * width, 0.5 * width
    tris = []
    for k in range(n):
        a0, a1 = th[k], th[k + 1]
        p = [(radius * np.cos(a), y, radius * np.sin(a)) for a in (a0, a1) for y in (y0, y1)]
        tris += [(p[0], p[2], p[3]), (p[0], p[3], p[1])]
        for y in (y0, y1):  # side disks as fans
            tris.append(((0.0, y, 0.0), (radius * np.cos(a0), y, radius * np.sin(a0)),
                         (radius * np.cos(a1), y, radius * np.sin(a1))))
    for g in range(grousers):
        a = 2 * np.pi * g / grousers
        c, s_ = np.cos(a), np.sin(a)
        r0, r1 = radius, radius + grouser_h
        q = [(r * c, y, r * s_) for r in (r0, r1) for y in (y0, y1)]
        tris += [(q[0], q[2], q[3]), (q[0], q[3], q[1])]
    return np.array(tris, dtype=np.float64)
