"""Digital-simulant (DS) clump templates and materials — seeded input data only.

This module builds the *inputs* both implementations consume (template geometry,
mass, principal inertia, material table).  It contains none of the method's
per-step arithmetic (no contact, force or integration code): that lives in
`oracle/` (CPU checker) and in `paper_2307_03445_b200/csrc/` (the CUDA product),
which share nothing but what this module hands them.

Sources
-------
* PAPER.md:188-199 (Table 1): seven DS types, bounding size D, component radius r,
  weight %, and the material E=1e9 Pa, nu=0.3, mu_s=0.4, CoR=0.5.
* PAPER.md:169 (Sec. 3): types 1-2 are six overlapping spheres forming a flat
  triangle, types 3-7 three spheres, all with 120-degree rotational symmetry; size
  is the bounding-sphere diameter.
* Geometry reading (DESIGN.md "readings" R22): three
  spheres on a circle of radius D/2 - r at 0/120/240 deg; types 1-2 add three
  fillers on a circle of half that radius at 60/180/300 deg.  All coplanar (z=0).
* Mass/inertia are of the geometric UNION, computed here by a
  midpoint voxel rule at the template's own resolution; grain density 2600 kg/m^3
  (SURVEY.md O19 — unpinned by the paper, an input to both sides).
* Number fractions: Table 1 weight fractions divided by the sum-of-sphere volume
  of each type.  This reading reproduces the paper's
  base-patch ratio 13,993,536 / 4,571,136 = 3.06128 spheres per clump.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

# ---------------------------------------------------------------- Table 1
DS_SIZE_MM = np.array([21.0, 11.4, 6.6, 4.5, 3.0, 2.75, 2.5])
DS_RADIUS_MM = np.array([3.6, 1.95, 1.81, 1.24, 0.82, 0.75, 0.7])
DS_WEIGHT_PCT = np.array([17.0, 21.0, 14.0, 19.0, 16.0, 5.0, 8.0])
DS_NCOMP = np.array([6, 6, 3, 3, 3, 3, 3])
GRAIN_DENSITY = 2600.0  # kg/m^3; not fixed by the paper

# Table 1 caption material, and the C4 per-sphere material set.
M0 = (1.0e9, 0.3, 0.4, 0.5)  # (E [Pa], nu, mu, CoR) — P:198
C4_MATERIALS = [
    M0,
    (5.0e8, 0.25, 0.3, 0.6),
    (2.0e9, 0.35, 0.5, 0.4),
    (1.0e9, 0.3, 0.6, 0.7),
]


@dataclass
class Template:
    """A clump template in its principal body frame (COM at origin)."""

    offsets: np.ndarray  # (n, 3) body-frame sphere centres [m]
    radius: np.ndarray  # (n,) [m]
    material: np.ndarray  # (n,) int32 material ids
    mass: float  # [kg]
    inertia: np.ndarray  # (3,) principal moments [kg m^2]
    name: str = ""

    @property
    def n_comp(self) -> int:
        return int(self.radius.shape[0])

    @property
    def bounding_radius(self) -> float:
        return float(np.max(np.linalg.norm(self.offsets, axis=1) + self.radius))


def ds_offsets(type_index: int, scale: float = 1.0, dilation: float = 1.0) -> tuple[np.ndarray, float]:
    """Body-frame component centres [m] and radius [m] of DS type `type_index` (0-based).

    Construction per SPEC.md:398 (reading R22); `dilation` scales centre distances
    only (P:540 dilated clumps; not used by the configs).
    """
    D = DS_SIZE_MM[type_index] * 1e-3 * scale
    r = DS_RADIUS_MM[type_index] * 1e-3 * scale
    d_out = (D / 2.0 - r) * dilation
    pts = []
    for k in range(3):
        a = math.radians(120.0 * k)
        pts.append((d_out * math.cos(a), d_out * math.sin(a), 0.0))
    if DS_NCOMP[type_index] == 6:
        for k in range(3):
            a = math.radians(60.0 + 120.0 * k)
            pts.append((0.5 * d_out * math.cos(a), 0.5 * d_out * math.sin(a), 0.0))
    return np.array(pts, dtype=np.float64), r


def union_mass_inertia(offsets: np.ndarray, radius: np.ndarray, density: float,
                       vox_per_rmin: int = 24) -> tuple[float, np.ndarray, np.ndarray]:
    """Mass, COM and inertia tensor (about COM) of a union of spheres, midpoint voxels.

    Voxel grid is centred on the origin so symmetric bodies get a symmetric grid.
    """
    pitch = float(np.min(radius)) / vox_per_rmin
    lo = np.min(offsets - radius[:, None], axis=0)
    hi = np.max(offsets + radius[:, None], axis=0)
    ext = np.maximum(np.abs(lo), np.abs(hi))
    n = np.ceil(ext / pitch).astype(int)
    axes = [(np.arange(-n[d], n[d]) + 0.5) * pitch for d in range(3)]
    mass = 0.0
    first = np.zeros(3)
    second = np.zeros((3, 3))
    dv = pitch ** 3
    # slice along z to bound memory
    X, Y = np.meshgrid(axes[0], axes[1], indexing="ij")
    for z in axes[2]:
        inside = np.zeros(X.shape, dtype=bool)
        for o, r in zip(offsets, radius):
            inside |= (X - o[0]) ** 2 + (Y - o[1]) ** 2 + (z - o[2]) ** 2 <= r * r
        if not inside.any():
            continue
        xs, ys = X[inside], Y[inside]
        zs = np.full(xs.shape, z)
        m = density * dv
        mass += m * xs.size
        P = np.stack([xs, ys, zs])
        first += m * P.sum(axis=1)
        second += m * (P @ P.T)
    com = first / mass
    # inertia about COM: I = sum m (|p|^2 E - p p^T), shifted by parallel axis
    S = second - mass * np.outer(com, com)
    inertia = np.trace(S) * np.eye(3) - S
    return mass, com, inertia


def ds_template(type_index: int, material: int | list[int] = 0, density: float = GRAIN_DENSITY,
                scale: float = 1.0) -> Template:
    """DS type `type_index` (0-based; paper type = index+1) with principal inertia.

    The construction is symmetric: COM is the origin and the plane z=0 is a
    principal plane with isotropic in-plane inertia (120-deg symmetry), so the
    construction frame is the principal frame.  Voxel noise in the in-plane pair
    is averaged out to keep that symmetry exact.
    """
    offs, r = ds_offsets(type_index, scale)
    n = offs.shape[0]
    rad = np.full(n, r)
    mats = np.array(material if isinstance(material, (list, tuple, np.ndarray)) else [material] * n,
                    dtype=np.int32)
    assert mats.shape == (n,)
    mass, com, I = union_mass_inertia(offs, rad, density)
    ip = 0.5 * (I[0, 0] + I[1, 1])
    return Template(offsets=offs, radius=rad, material=mats, mass=mass,
                    inertia=np.array([ip, ip, I[2, 2]]), name=f"DS{type_index + 1}")


def sphere_template(radius: float, material: int = 0, density: float = GRAIN_DENSITY) -> Template:
    """Single-sphere clump with analytic mass and inertia (P:517 monodisperse case)."""
    m = density * 4.0 / 3.0 * math.pi * radius ** 3
    i = 0.4 * m * radius ** 2
    return Template(offsets=np.zeros((1, 3)), radius=np.array([radius]),
                    material=np.array([material], dtype=np.int32), mass=m,
                    inertia=np.array([i, i, i]), name=f"sphere{radius * 1e3:g}mm")


def ds_number_fractions() -> np.ndarray:
    """Table-1 weight fractions -> number fractions via sum-of-sphere volumes (fact 0.1-5)."""
    vol = DS_NCOMP * (4.0 / 3.0 * math.pi * DS_RADIUS_MM ** 3)
    w = DS_WEIGHT_PCT / DS_WEIGHT_PCT.sum()
    f = w / vol
    return f / f.sum()


def ds_type_counts(n_clumps: int) -> np.ndarray:
    """Deterministic quota of clumps per DS type (largest-remainder rounding)."""
    f = ds_number_fractions() * n_clumps
    base = np.floor(f).astype(np.int64)
    rem = n_clumps - int(base.sum())
    order = np.argsort(-(f - base), kind="stable")
    base[order[:rem]] += 1
    return base


def ds_templates(per_component_materials: bool = False, density: float = GRAIN_DENSITY) -> list[Template]:
    """All seven DS templates.  With `per_component_materials`, component k of each
    template gets material k mod 4."""
    out = []
    for t in range(7):
        n = int(DS_NCOMP[t])
        mats = [k % 4 for k in range(n)] if per_component_materials else [0] * n
        out.append(ds_template(t, mats, density))
    return out
