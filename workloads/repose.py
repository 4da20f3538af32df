"""Repose-angle scene: settled DS material poured through a
funnel mesh onto a floor — inputs only, no method arithmetic.

P:277: "the initial sample is prepared by taking a cylindrical portion out of a DS patch, making
three extra copies, and then translating everything into a funnel defined via a mesh ... The
material flows through the funnel under gravity."  The paper's sample has 731,060 clumps; this
one is a scaled-down copy of the same recipe: `copies` cylinders of radius `radius` cut from the
oracle-settled 30 mm patch, placed side by side above a conical funnel whose opening is wide
enough for the 21 mm type-1 clumps, released from rest above the floor plane z = 0.
"""
from __future__ import annotations

import math

import numpy as np

from .beds import load_patch
from .ds import M0
from .scenes import Mesh, Plane, Scene, mesh_funnel


def repose_scene(copies: int = 4, radius: float = 14e-3, r_top: float = 0.07, r_open: float = 0.03,
                 funnel_h: float = 0.05, funnel_z: float = 0.08, h: float = 1e-6) -> Scene:
    p = load_patch()
    side_x = max(pl.point[0] for pl in p.planes if pl.normal[0] < 0)
    side_y = max(pl.point[1] for pl in p.planes if pl.normal[1] < 0)
    cx, cy = 0.5 * side_x, 0.5 * side_y
    sel = np.nonzero(np.hypot(p.pos[:, 0] - cx, p.pos[:, 1] - cy) < radius)[0]
    col = p.subset(sel)
    z0 = float(col.pos[:, 2].min())
    # column axes on a circle, neighbours apart by 2 radius + 12 mm (a 21 mm type-1 clump cut by its
    # COM sticks out of its column by up to 10.5 mm); the columns stand just above the funnel
    if copies <= 6:
        ring = (2 * radius + 12e-3) / (2 * math.sin(math.pi / copies)) if copies > 1 else 0.0
        offs = [(ring * math.cos(2 * math.pi * k / copies), ring * math.sin(2 * math.pi * k / copies))
                for k in range(copies)]
    else:  # a square grid of columns
        m = math.ceil(math.sqrt(copies))
        pitch = 2 * radius + 12e-3
        offs = [((i - (m - 1) / 2) * pitch, (j - (m - 1) / 2) * pitch) for i in range(m) for j in range(m)][:copies]
    base = funnel_z + funnel_h + 2e-3
    pos, quat, vel, om, tid = [], [], [], [], []
    for (ox, oy) in offs:
        P = col.pos.copy()
        P[:, 0] += ox - cx
        P[:, 1] += oy - cy
        P[:, 2] += base - z0
        pos.append(P)
        quat.append(col.quat)
        vel.append(np.zeros_like(col.vel))
        om.append(np.zeros_like(col.omega))
        tid.append(col.tid)
    pos, quat = np.concatenate(pos), np.concatenate(quat)
    n = pos.shape[0]
    # floor z = 0; side walls far outside the pile keep the odd clump that rolls away in the domain
    L = 0.24
    planes = [Plane((0.0, 0.0, 0.0), (0.0, 0.0, 1.0), 0), Plane((-L, 0.0, 0.0), (1.0, 0.0, 0.0), 0),
              Plane((L, 0.0, 0.0), (-1.0, 0.0, 0.0), 0), Plane((0.0, -L, 0.0), (0.0, 1.0, 0.0), 0),
              Plane((0.0, L, 0.0), (0.0, -1.0, 0.0), 0)]
    s = Scene(materials=np.array([M0]), templates=p.templates, planes=planes,
              h=h, gravity=np.array([0.0, 0.0, -9.81]), domain_lo=np.array([-0.25, -0.25, -0.01]),
              domain_hi=np.array([0.25, 0.25, float(pos[:, 2].max()) + 0.05]),
              gid=np.arange(n, dtype=np.int64), tid=np.concatenate(tid).astype(np.int32), pos=pos, quat=quat,
              vel=np.concatenate(vel), omega=np.concatenate(om), name=f"repose-{n}")
    s.meshes = [Mesh(mesh_funnel(r_top, r_open, funnel_h, 48), 0, pos=(0.0, 0.0, funnel_z))]
    return s


def pile_angle(pos, bound_r, axis=(0.0, 0.0), z_max=None, dr=2e-3):
    """Angle of the pile's free surface: in rings of width dr about the axis, the surface height is
    the highest top (COM z + bounding radius) of the clumps below z_max; a line is fitted to the
    heights of the rings between 20% and 80% of the pile radius (the cap and the toe excluded)."""
    rho = np.hypot(pos[:, 0] - axis[0], pos[:, 1] - axis[1])
    top = pos[:, 2] + bound_r
    keep = np.ones(len(rho), bool) if z_max is None else pos[:, 2] < z_max
    rho, top = rho[keep], top[keep]
    edges = np.arange(0.0, rho.max() + dr, dr)
    idx = np.digitize(rho, edges) - 1
    surf = np.full(len(edges) - 1, np.nan)
    for k in range(len(edges) - 1):
        m = idx == k
        if m.sum() >= 3:
            surf[k] = np.sort(top[m])[-2]  # second highest: robust to a lone clump on top
    r_mid = 0.5 * (edges[1:] + edges[:-1])
    ok = ~np.isnan(surf)
    # pile radius: the outermost ring still holding a 5 mm thick layer
    thick = ok & (surf > 5e-3)
    R = r_mid[thick].max() if thick.any() else r_mid[ok].max()
    fit = ok & (r_mid >= 0.2 * R) & (r_mid <= 0.8 * R)
    slope, icpt = np.polyfit(r_mid[fit], surf[fit], 1)
    return dict(angle_deg=float(math.degrees(math.atan(-slope))), radius_m=float(R), height_m=float(icpt),
                profile=[(float(a), float(b)) for a, b in zip(r_mid[ok], surf[ok])])
