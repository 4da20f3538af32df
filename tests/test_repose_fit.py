"""The repose-angle measurement of NEXT-4 (tools/repose_c3.py, workloads.repose.pile_angle) on
synthetic piles of known angle: clump centres filling a cone of slope theta (P:277's quantity),
so the fitted free-surface angle is pinned independently of any simulation."""
import importlib.util
import math
import os

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _tool():
    spec = importlib.util.spec_from_file_location("repose_c3", os.path.join(ROOT, "tools", "repose_c3.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def _cone(theta_deg, n=60_000, R=0.15, seed=0, top_r=2e-3):
    """n centres uniform in a solid cone of base radius R and slope theta, apex on the axis, their
    bounding spheres touching the cone surface from below (top = centre z + top_r)."""
    rng = np.random.default_rng(seed)
    H = R * math.tan(math.radians(theta_deg))
    pts = []
    while sum(len(p) for p in pts) < n:
        xy = rng.uniform(-R, R, size=(4 * n, 2))
        z = rng.uniform(0.0, H, size=4 * n)
        rho = np.hypot(xy[:, 0], xy[:, 1])
        surf = (R - rho) * math.tan(math.radians(theta_deg))
        ok = (rho < R) & (z + top_r <= surf)
        pts.append(np.column_stack([xy[ok], z[ok]]))
    return np.concatenate(pts)[:n] + np.array([0.31, -0.07, 0.0])  # off-origin: the centre is found


@pytest.mark.parametrize("theta", [25.0, 30.0, 35.0])
def test_fit_angles_recovers_a_cone(theta):
    tool = _tool()
    pos = _cone(theta)
    r_mid, surf, _ = tool.surface_profile(pos, 2e-3)
    R, fits = tool.fit_angles(r_mid, surf)
    assert len(fits) >= 4
    for k, a in fits.items():
        assert abs(a - theta) < 1.0, (k, a)
    assert abs(R - 0.15) < 0.02


@pytest.mark.parametrize("theta", [25.0, 30.0, 35.0])
def test_pile_angle_recovers_a_cone(theta):
    from workloads.repose import pile_angle

    pos = _cone(theta, seed=1)
    out = pile_angle(pos, 2e-3, axis=(0.31, -0.07))
    assert abs(out["angle_deg"] - theta) < 1.0
