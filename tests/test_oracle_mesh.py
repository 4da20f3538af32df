"""Pins of the oracle's kinematic triangle meshes (NEXT-3; P:277 cone penetrometer, P:344 wheel;
SPEC S:241-262 sphere_triangle_contact / body_wrench / advance_boundary).

Each test checks the oracle against something other than itself: an independent closest-point
construction, the analytic plane it must reproduce, closed-form collisions against a moving
wall and a moving belt, static equilibrium, symmetry, and the exact rotation of a spinning
mesh.  DESIGN.md R25-R27 state the readings.
"""
import math

import numpy as np
import pytest

import oracle
import workloads as w
from workloads.scenes import Mesh, mesh_cone, mesh_rect, sphere_on_mesh

RHO = 2600.0
E_STAR = 1e9 / (2 * (1 - 0.3 ** 2))  # M0 on M0


def _rest_delta(r=1e-3):
    """Static Hertz penetration of a resting sphere: (4/3) E* sqrt(r) delta^1.5 = m g."""
    m = RHO * 4.0 / 3.0 * math.pi * r ** 3
    return (m * 9.81 / (4.0 / 3.0 * E_STAR * math.sqrt(r))) ** (2.0 / 3.0)


def _independent_closest(p, a, b, c):
    """Projection onto the plane (barycentric by least squares); if outside, the best of the three
    clamped segment projections.  Shares nothing with the Voronoi-region construction."""
    A = np.stack([b - a, c - a], axis=1)
    st, *_ = np.linalg.lstsq(A, p - a, rcond=None)
    if st[0] >= 0 and st[1] >= 0 and st[0] + st[1] <= 1:
        return a + A @ st, "face"
    best, kind = None, None
    for (u, v, name) in ((a, b, "ab"), (a, c, "ac"), (b, c, "bc")):
        t = np.clip(np.dot(p - u, v - u) / np.dot(v - u, v - u), 0.0, 1.0)
        q = u + t * (v - u)
        if best is None or np.linalg.norm(p - q) < np.linalg.norm(p - best):
            best, kind = q, ("v" if t in (0.0, 1.0) else name)
    return best, kind


def test_closest_point_matches_independent_projection():
    rng = np.random.default_rng(7)
    regions = set()
    for _ in range(3000):
        a, b, c = rng.normal(size=(3, 3)) * 1e-3
        p = rng.normal(size=3) * 2e-3
        q, reg = oracle.closest_on_triangle(p, a, b, c)
        qi, kind = _independent_closest(p, a, b, c)
        assert np.linalg.norm(q - qi) <= 1e-12 + 1e-9 * np.linalg.norm(p - qi), (p, a, b, c)
        regions.add(reg)
        if kind == "face":
            assert reg == 0
        elif kind in ("ab", "ac", "bc"):
            assert reg == {"ab": 1, "ac": 2, "bc": 3}[kind]
    assert regions == set(range(7))  # every Voronoi region was exercised


@pytest.mark.parametrize("at", [(0.3e-3, -0.2e-3), (0.0, 0.0), (2.5e-3, 0.0), (1.25e-3, -1.25e-3)])
def test_sphere_on_mesh_square_equals_analytic_plane(at):
    """A sphere hitting a flat mesh square (face, shared vertex of 6 triangles, shared edge, a
    diagonal) moves exactly like one hitting the analytic plane z = 0: one contact per feature
    (R26) and the flat-wall limit R_bar = r, m_bar = M."""
    kw = dict(drop=2e-6, v0=(0.0, 0.0, -0.3), at=at)
    m = oracle.Oracle(sphere_on_mesh(**kw))
    p = oracle.Oracle(sphere_on_mesh(with_plane=True, **kw))
    for _ in range(6):
        m.step(500)
        p.step(500)
        sm, sp = m.state(), p.state()
        # identical up to rounding: the mesh normal (c - q)/|c - q| carries ~1e-16 tangential
        # noise from the closest-point arithmetic, the plane's normal is exact
        for k, atol in (("pos", 1e-15), ("vel", 1e-12), ("omega", 1e-9)):
            assert np.allclose(sm[k], sp[k], rtol=1e-12, atol=atol), k
    assert abs(m.state()["vel"][0, 2]) < 0.3  # it bounced (CoR 0.5) and is settling


def test_head_on_against_moving_mesh_wall_restitution():
    """g = 0, sphere at rest; the mesh plate rises at V: in the plate frame a head-on wall impact
    at speed V, so the sphere leaves at (1 + e) V with e = CoR (fact 0.1-1), and the plate moves
    exactly V per step (advance_boundary)."""
    V = 0.5
    s = sphere_on_mesh(drop=1e-6, g=(0.0, 0.0, 0.0), mesh_vel=(0.0, 0.0, V), h=5e-7)
    o = oracle.Oracle(s)
    o.step(2000)  # contact lasts ~80 steps
    vz = o.state()["vel"][0, 2]
    e = (vz - V) / V
    assert abs(e - 0.5) < 1e-3, e
    X = o.mesh(0)["pos"]
    assert abs(X[2] - V * 5e-7 * 2000) < 1e-15


def test_sphere_dragged_by_moving_belt_reaches_two_sevenths():
    """A resting sphere on a plate sliding at V (friction sees the boundary's velocity):
    kinetic friction accelerates the centre at mu g and spins it at 5 mu g / (2 r) until the
    contact point stops slipping, at v = (2/7) V whatever mu is."""
    V = 0.05
    s = sphere_on_mesh(drop=-_rest_delta(), mesh_vel=(V, 0.0, 0.0))
    s.meshes[0].verts = mesh_rect(0.5, 0.01, 1, 1)  # long enough for the belt to pass under it
    o = oracle.Oracle(s)
    o.step(12_000)  # slip ends after V / (3.5 mu g) = 3.6 ms
    vx = o.state()["vel"][0, 0]
    assert abs(vx - 2.0 / 7.0 * V) < 0.01 * V, vx


def test_resting_weight_and_zero_torque_of_symmetric_pair():
    """Static equilibrium: the wrench on a plate under two resting spheres placed symmetrically
    about its reference point is (0, 0, -2 m g) within 1% with zero torque."""
    r = 1e-3
    s = sphere_on_mesh()
    z = r - _rest_delta(r)
    s.pos = np.array([[2e-3, 1e-3, z], [-2e-3, -1e-3, z]])
    s.gid, s.tid = np.array([0, 1]), np.array([0, 0], np.int32)
    s.quat = np.tile([1.0, 0, 0, 0], (2, 1))
    s.vel, s.omega = np.zeros((2, 3)), np.zeros((2, 3))
    o = oracle.Oracle(s)
    o.step(4000)
    m = RHO * 4.0 / 3.0 * math.pi * r ** 3
    F, T = o.mesh(0)["force"], o.mesh(0)["torque"]
    assert abs(F[2] + 2 * m * 9.81) < 0.01 * 2 * m * 9.81, F
    assert abs(F[0]) + abs(F[1]) < 1e-9 * m * 9.81
    assert np.abs(T).max() <= 1e-12 * 2e-3 * m * 9.81 + 1e-20, T


def test_spinning_mesh_pose_is_the_exact_rotation():
    """advance_boundary with angular velocity w: after n steps the pose is the rotation by n h |w|
    (to rounding), and the world vertices follow it."""
    wz = 50.0
    s = sphere_on_mesh(drop=5e-3, g=(0.0, 0.0, 0.0), mesh_omega=(0.0, 0.0, wz))
    o = oracle.Oracle(s)
    n = 4000
    o.step(n)
    th = n * s.h * wz
    q = o.mesh(0)["quat"]
    assert np.allclose(q, [math.cos(th / 2), 0, 0, math.sin(th / 2)], atol=1e-13), q


def test_cone_contact_set_matches_brute_force():
    """Candidate sphere-triangle pairs on a faceted cone (the P:277 penetrometer tip) equal an
    independent numpy enumeration |c - closest|^2 <= (r + margin)^2 with the independent
    projection above; keys are (sphere key, INT64_MAX - 16 - triangle)."""
    rng = np.random.default_rng(11)
    cone = mesh_cone(0.01 * math.tan(math.radians(30)), 0.01, 16)
    scene = w.random_spheres(5, 400, box=0.012) if hasattr(w, "random_spheres") else None
    assert scene is not None
    scene.planes = []
    scene.pos[:, :2] -= 0.006
    scene.pos[:, 2] -= 0.001
    scene.meshes = [Mesh(cone, 0, pos=(0.0, 0.0, 0.0))]
    scene.gravity = np.zeros(3)
    scene.domain_lo, scene.domain_hi = np.full(3, -0.02), np.full(3, 0.03)
    margin = 0.2e-3
    o = oracle.Oracle(scene, margin=margin)
    o.step(1)
    c = o.contacts()
    mesh_keys = c["key_b"] > np.iinfo(np.int64).max - 16 - 10_000
    got = sorted(zip(c["key_a"][mesh_keys & (c["key_b"] <= np.iinfo(np.int64).max - 16)].tolist(),
                     c["key_b"][mesh_keys & (c["key_b"] <= np.iinfo(np.int64).max - 16)].tolist()))
    want = []
    rad = np.array([scene.templates[t].radius[0] for t in scene.tid])
    for k in range(scene.n_clumps):
        p = scene.pos[k]
        for t, (a, b, cc) in enumerate(cone):
            q, _ = _independent_closest(p, a, b, cc)
            d2 = np.sum((p - q) ** 2)
            s_ = rad[k] + margin
            if d2 <= s_ * s_ * (1 - 1e-12):
                want.append((int(scene.gid[k]) * 64, np.iinfo(np.int64).max - 16 - t))
            elif d2 <= s_ * s_ * (1 + 1e-12):
                pytest.skip("a pair within rounding of the threshold")
    assert len(want) > 20
    assert got == sorted(want)
