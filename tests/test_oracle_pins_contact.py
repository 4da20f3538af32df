"""Pins of the oracle's contact-level readings that the round-1 pins left free (no GPU).

A mutation test of the oracle (tools/mutate_oracle.py) showed that these
readings could be changed without failing any pin:
  * the tangential damping c_t = 2 sqrt(5/6) beta sqrt(k_t m)   (Eq. 1b; O2)
  * the contact point at the middle of the overlap, for r_a != r_b and for walls
                                                             ("mutual contact point"; O6)
  * the Eq. 3c branch taken on the trial force *with* damping    (O7)
Each test below is a closed form of rigid-body / oscillator mechanics that one of those
readings implies; a plausible mistake in the corresponding oracle line fails it.
"""
import math

import numpy as np
import pytest
from scipy.spatial.transform import Rotation

import oracle
import workloads as w
from workloads import scenes

G = 9.81


def _estar(E, nu):
    # same material on both sides: 1/E* = 2 (1 - nu^2)/E, 1/G* = 2 * 2 (2 - nu)(1 + nu)/E
    return E / (2 * (1 - nu * nu)), E / (4 * (2 - nu) * (1 + nu))


def _beta(cor):
    le = math.log(cor)
    return -le / math.sqrt(le * le + math.pi ** 2)


def _resting(mat, r, g_vec, h, v0=(0.0, 0.0, 0.0), mesh=False, at=(0.0, 0.0)):
    """One sphere of radius r resting on z = 0 (analytic plane or a large mesh square) at its
    static Hertz penetration under the normal load m g_n: (4/3) E* sqrt(r) d0^1.5 = m g_n."""
    t = w.sphere_template(r, 0)
    Es, _ = _estar(mat[0], mat[1])
    gn = -g_vec[2]
    d0 = (t.mass * gn / (4.0 / 3.0 * Es * math.sqrt(r))) ** (2.0 / 3.0)
    s = w.Scene(materials=np.array([mat]), templates=[t], planes=[], h=h, gravity=np.array(g_vec, float),
                domain_lo=np.array([-0.5, -0.5, -0.1]), domain_hi=np.array([0.5, 0.5, 0.1]),
                gid=np.array([3], np.int64), tid=np.array([0], np.int32),
                pos=np.array([[at[0], at[1], r - d0]]), quat=np.array([[1.0, 0, 0, 0]]),
                vel=np.array([v0], float), omega=np.zeros((1, 3)))
    if mesh:
        s.meshes = [scenes.Mesh(scenes.mesh_rect(0.8, 0.8, 2, 2), 0)]
    else:
        s.planes = [w.Plane((0.0, 0.0, 0.0), (0.0, 0.0, 1.0), 0)]
    return s, t, d0


# ---------------------------------------------------------------- c_t (Eq. 1b)
def test_tangential_damping_log_decrement():
    """A sphere resting on a plane, kicked tangentially inside the stick regime: the contact
    point's tangential displacement x obeys m_eff x'' = -k_t x - c_t x' with
    1/m_eff = 1/m + rho^2/I (translation + rolling about the lever arm rho = r - delta/2),
    so successive maxima of u_t shrink by exp(-2 pi zeta / sqrt(1 - zeta^2)) with
    zeta = c_t / (2 sqrt(k_t m_eff)) and the period is 2 pi / (omega_n sqrt(1 - zeta^2)).
    With c_t of reading O2 (m-bar = M for a wall): zeta = sqrt(5/6) beta sqrt(M/m_eff)."""
    mat = (1e9, 0.3, 0.9, 0.5)  # mu = 0.9 keeps the kick well inside the cap
    r = 1e-3
    Es, Gs = _estar(mat[0], mat[1])
    t = w.sphere_template(r)
    m, I = t.mass, t.inertia[0]
    d0 = (m * G / (4.0 / 3.0 * Es * math.sqrt(r))) ** (2.0 / 3.0)
    rho = r - 0.5 * d0
    m_eff = 1.0 / (1.0 / m + rho * rho / I)
    k_t = 8.0 * Gs * math.sqrt(r * d0)
    zeta = math.sqrt(5.0 / 6.0) * _beta(mat[3]) * math.sqrt(m / m_eff)
    wn = math.sqrt(k_t / m_eff)
    T = 2 * math.pi / (wn * math.sqrt(1 - zeta * zeta))
    h = T / 2000
    s, _, _ = _resting(mat, r, (0.0, 0.0, -G), h, v0=(2e-5, 0.0, 0.0))
    o = oracle.Oracle(s)
    n = int(3.3 * T / h)
    u = np.zeros(n)
    for k in range(n):
        o.step(1)
        c = o.contacts()
        assert len(c["key_a"]) == 1 and c["delta"][0] > 0
        u[k] = c["u_t"][0, 0]
    # maxima of u (the first one sits a quarter period in; then one per period)
    pk = [k for k in range(1, n - 1) if u[k] > u[k - 1] and u[k] >= u[k + 1] and u[k] > 0]
    assert len(pk) >= 3
    ratio = u[pk[1]] / u[pk[0]]
    want = math.exp(-2 * math.pi * zeta / math.sqrt(1 - zeta * zeta))
    assert ratio == pytest.approx(want, rel=5e-3), (ratio, want)
    assert u[pk[2]] / u[pk[1]] == pytest.approx(want, rel=5e-3)
    assert (pk[1] - pk[0]) * h == pytest.approx(T, rel=2e-3)
    # test power: c_t from S_n (sqrt(S_n m) instead of sqrt(k_t m)) moves zeta by ~10%, and
    # c_t = 0 gives ratio 1
    zeta_sn = zeta * math.sqrt(2 * Es / (8 * Gs))
    assert abs(math.exp(-2 * math.pi * zeta_sn / math.sqrt(1 - zeta_sn ** 2)) / want - 1) > 0.05


# ---------------------------------------------------------------- wall contact point (O6)
@pytest.mark.parametrize("boundary", ["plane", "mesh"])
def test_soft_sphere_rolls_about_the_middle_of_the_overlap(boundary):
    """Rolling without slip on an incline about the contact point p = c - (r - delta/2) n_w
    (the middle of the overlap, reading O6) gives a = g sin(alpha) / (1 + I / (m rho^2)) with
    rho = r - delta/2.  A soft material (delta/r = 0.1) separates it from rho = r (the sphere
    surface) by 3%.  The incline is a tilted gravity vector."""
    r, alpha, nu = 1e-3, math.radians(20.0), 0.3
    t = w.sphere_template(r)
    gn = G * math.cos(alpha)
    d_target = 0.1 * r
    Es = t.mass * gn / (4.0 / 3.0 * math.sqrt(r) * d_target ** 1.5)
    mat = (Es * 2 * (1 - nu * nu), nu, 0.6, 0.5)
    g_vec = (G * math.sin(alpha), 0.0, -gn)
    h = 1e-5
    s, _, d0 = _resting(mat, r, g_vec, h, mesh=(boundary == "mesh"), at=(-0.3, 0.0))
    assert d0 == pytest.approx(d_target, rel=1e-9)
    o = oracle.Oracle(s)
    ts, vs = [], []
    for k in range(60):
        o.step(500)
        ts.append((k + 1) * 500 * h)
        vs.append(o.state()["vel"][0, 0])
    ts, vs = np.array(ts), np.array(vs)
    sel = ts >= 0.1
    a = np.polyfit(ts[sel], vs[sel], 1)[0]
    I = t.inertia[0]
    rho = r - 0.5 * d0
    want = G * math.sin(alpha) / (1 + I / (t.mass * rho * rho))
    surface = G * math.sin(alpha) / (1 + I / (t.mass * r * r))
    assert abs(surface / want - 1) > 0.02  # the test can tell the two points apart
    assert a == pytest.approx(want, rel=3e-3), (a, want, surface)


# ---------------------------------------------------------------- polydisperse contact point (O6)
@pytest.mark.parametrize("small_first", [True, False])
def test_oblique_impact_spin_follows_each_spheres_own_lever_arm(small_first):
    """Frictional oblique impact of a small (r_a) and a large (r_b = 3 r_a) sphere, g = 0.  The
    contact point is on both surfaces, at distance rho_a = r_a - delta/2 from c_a and
    rho_b = r_b - delta/2 from c_b (p = (c_a + c_b)/2 + (r_a - r_b)/2 n).
    Each sphere's torque is rho n x (its contact force), so its spin angular momentum change is
    L_a = rho_a n x dP_a and L_b = -rho_b n x dP_b: with n ~ +x (a -> b) and the tangential
    impulse along y, L_z / dP_y = rho_a for a and -rho_b for b.  Putting p at the midpoint of
    the centres instead would give (r_a + r_b)/2 for both (x2 and x2/3 off).  Both key orders
    are run so the (r_a - r_b) sign is exercised with the small sphere as a and as b."""
    ra, rb = 0.5e-3, 1.5e-3
    ta, tb = w.sphere_template(ra), w.sphere_template(rb)
    gid = np.array([0, 1] if small_first else [1, 0], np.int64)
    s = w.Scene(materials=np.array([w.M0]), templates=[ta, tb], planes=[], h=2e-8, gravity=np.zeros(3),
                domain_lo=np.full(3, -0.02), domain_hi=np.full(3, 0.02), gid=gid, tid=np.array([0, 1], np.int32),
                pos=np.array([[0.0, 0.0, 0.0], [ra + rb, 0.0, 0.0]]), quat=np.array([[1.0, 0, 0, 0]] * 2),
                vel=np.array([[0.2, 0.08, 0.0], [0.0, 0.0, 0.0]]), omega=np.zeros((2, 3)))
    o = oracle.Oracle(s)
    st0 = o.state()
    touched, dmax = False, 0.0
    for _ in range(20000):
        o.step(10)
        c = o.contacts()
        live = c["delta"] > 0
        touched |= bool(live.any())
        if live.any():
            dmax = max(dmax, float(c["delta"].max()))
        if touched and not live.any():
            break
    assert touched and not live.any()
    st = o.state()
    res = []
    for k, t in ((0, ta), (1, tb)):
        dP = t.mass * (st["vel"][k] - st0["vel"][k])
        R = Rotation.from_quat(st["quat"][k, [1, 2, 3, 0]]).as_matrix()
        L = R @ (t.inertia * st["omega"][k])
        assert abs(dP[1]) > 0.05 * abs(dP[0])  # a real tangential impulse (friction acted)
        res.append(L[2] / dP[1])
    # lever arms r - delta/2 (delta/2 <= 0.1% of r here), up to the turn of n during the
    # contact (n_y dP_x enters L_z: 0.3% here); the midpoint of the centres would give 2 r_a
    # and -(2/3) r_b
    assert res[0] == pytest.approx(ra, rel=1e-2), (res, ra, dmax)
    assert res[1] == pytest.approx(-rb, rel=1e-2), (res, rb, dmax)


# ---------------------------------------------------------------- Eq. 3c branch (O7)
def test_kick_where_damping_alone_exceeds_the_cap_slides_at_mu_g():
    """A resting sphere is given a tangential speed v0 so large that c_t v0 > mu |F_n| while the
    first-step spring force k_t h v0 is below it.  Eq. 3c with the trial force
    including damping (reading O7) puts the contact in the sliding branch from the first step,
    so |F_t| <= mu |F_n| holds at every step and the sphere decelerates at exactly the
    kinetic rate: V(t) = v0 - mu g t, Omega(t) = 5 mu g t / (2 r)  (sliding sphere, Coulomb
    friction on a level plane).  Branching on the undamped spring force alone would keep it
    "stuck" and apply the full damped force, far above the cap."""
    mat = (1e9, 0.3, 0.4, 0.5)
    r, h, v0 = 1e-3, 1e-8, 0.05
    s, t, d0 = _resting(mat, r, (0.0, 0.0, -G), h, v0=(v0, 0.0, 0.0))
    Es, Gs = _estar(mat[0], mat[1])
    k_t = 8.0 * Gs * math.sqrt(r * d0)
    c_t = 2 * math.sqrt(5.0 / 6.0) * _beta(mat[3]) * math.sqrt(k_t * t.mass)
    cap = mat[2] * t.mass * G
    assert k_t * h * v0 < 0.8 * cap and c_t * v0 > 100 * cap  # the two trial forces straddle the cap
    o = oracle.Oracle(s)
    n = 2000
    for k in range(n):
        o.step(1)
        c = o.contacts()
        F, nn = c["force_b"][0], c["normal"][0]
        fn = (F @ nn) * nn
        ft = F - fn
        assert np.linalg.norm(ft) <= mat[2] * np.linalg.norm(fn) * (1 + 1e-9), k
    st = o.state()
    T = n * h
    assert st["vel"][0, 0] - v0 == pytest.approx(-mat[2] * G * T, rel=2e-3)
    assert st["omega"][0, 1] == pytest.approx(5 * mat[2] * G * T / (2 * r), rel=2e-3)
