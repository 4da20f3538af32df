"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle, element by element.

Bars (BASELINE.json north_star): bit-exact sorted contact-pair set on identical input
states; per-contact forces within 1e-5 relative; clump states within 1e-4 relative after
100 steps.  Plus the closed forms and invariants re-checked on the GPU, determinism,
checkpoint/resume and edge cases.
"""
import numpy as np
import pytest

import oracle
import workloads as w
from _parity import assert_forces_close, assert_same_contact_set, assert_states_close

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dem():
    import torch

    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_2307_03445_b200 as pkg

    pkg.load_library()
    return pkg


def _evolved_c1(steps=400):
    s = w.c1_box()
    o = oracle.Oracle(s, detect=1)
    o.step(steps)
    st = o.state()
    s.pos, s.quat, s.vel, s.omega = st["pos"], st["quat"], st["vel"], st["omega"]
    c = o.contacts()
    return s, (c["key_a"], c["key_b"], c["u_t"])


SCENES = {
    "random_spheres_2mat": lambda: (w.random_spheres(41, 600, box=0.03, n_mat=2), None),
    "random_clumps_c4mats": lambda: (w.random_clumps(42, 300, box=0.03), None),
    "big_and_small_clumps": lambda: (w.random_clumps(43, 120, box=0.02, types=[0, 1, 6]), None),
    "c1_after_400_oracle_steps": lambda: _evolved_c1(400),
    "multi_tile_24k_spheres": lambda: (w.random_clumps(44, 8000, box=0.08), None),
}


def _pair(dem, scene, hist=None, record=True, **kw):
    g = dem.system_from_scene(scene, record_contacts=record, **kw)
    o = oracle.Oracle(scene)
    if hist is not None:
        g.dem_set_contact_history(*hist)
        o.set_history(*hist)
    return g, o


@pytest.mark.parametrize("name", list(SCENES))
def test_one_step_contacts_forces_state(dem, name):
    scene, hist = SCENES[name]()
    g, o = _pair(dem, scene, hist)
    g.dem_step(1)
    o.step(1)
    cg, co = g.dem_get_contacts(), o.contacts()
    assert len(co["key_a"]) > 0
    assert_same_contact_set(cg, co)
    assert_forces_close(cg, co, scene)
    s0 = dict(pos=scene.pos, quat=scene.quat)
    assert_states_close(g.dem_get_state(), o.state(), s0)
    st = g.dem_get_stats()
    assert st["n_contacts"] == len(co["key_a"])


def test_seeded_history_both_branches(dem):
    """Forces with identical random u_t seeded through dem_set_contact_history (stick and slip)."""
    scene = w.random_clumps(45, 300, box=0.03)
    probe = oracle.Oracle(scene)
    probe.step(1)
    c = probe.contacts()
    rng = np.random.default_rng(0)
    ut = rng.normal(size=(len(c["key_a"]), 3)) * rng.choice([1e-9, 1e-6, 1e-4], size=(len(c["key_a"]), 1))
    hist = (c["key_a"], c["key_b"], ut)
    g, o = _pair(dem, scene, hist)
    g.dem_step(1)
    o.step(1)
    cg, co = g.dem_get_contacts(), o.contacts()
    assert_same_contact_set(cg, co)
    assert_forces_close(cg, co, scene)
    # both Coulomb branches were exercised
    fn = (co["force_b"] * co["normal"]).sum(1)[:, None] * co["normal"]
    ft = np.linalg.norm(co["force_b"] - fn, axis=1)
    mu_cap = 0.3 * np.linalg.norm(fn, axis=1)
    assert (ft < mu_cap * 0.99).sum() > 10 and (ft > mu_cap * 1.0 - 1e-12).sum() > 10


@pytest.mark.parametrize("name", ["c1_after_400_oracle_steps", "random_clumps_c4mats"])
def test_states_after_100_steps(dem, name):
    scene, hist = SCENES[name]()
    g, o = _pair(dem, scene, hist, record=False)
    g.dem_step(100)
    o.step(100)
    errs = assert_states_close(g.dem_get_state(), o.state(), dict(pos=scene.pos, quat=scene.quat))
    print(name, errs)


def test_c1_full_1000_steps(dem):
    """Config 1 as specified: 1,000 three-sphere clumps settling in a box, 1,000 steps."""
    scene = w.c1_box()
    g = dem.system_from_scene(scene, record_contacts=True)
    o = oracle.Oracle(scene, detect=1)
    g.dem_step(1000)
    o.step(1000)
    assert_same_contact_set(g.dem_get_contacts(), o.contacts())
    assert_states_close(g.dem_get_state(), o.state(), dict(pos=scene.pos, quat=scene.quat))


@pytest.mark.parametrize("v0", [0.1, 1.0])
@pytest.mark.parametrize("mats,cor", [((0, 0), 0.5), ((0, 1), 0.5), ((1, 1), 0.8)])
def test_gpu_restitution_closed_form(dem, v0, mats, cor):
    """C2: e = CoR_pair (fact 0.1-1) on the GPU path."""
    m = w.sphere_template(1e-3).mass
    Es = oracle.pair_params(w.MAT_A if mats[0] == 0 else w.MAT_B, w.MAT_A if mats[1] == 0 else w.MAT_B)["e_star"]
    tc = 3.21807 * (3 * (m / 2) / (4 * Es * np.sqrt(0.5e-3))) ** 0.4 * v0 ** -0.2
    scene = w.c2_head_on(v0=v0, mats=mats, h=tc / 200)
    g = dem.system_from_scene(scene)
    g.dem_step(1200)
    st = g.dem_get_state()
    e = (st["vel"][1, 0] - st["vel"][0, 0]) / v0
    assert e == pytest.approx(cor, abs=1e-3)


def test_gpu_wall_restitution(dem):
    m = w.sphere_template(1e-3).mass
    Es = oracle.pair_params(w.MAT_A, w.MAT_B)["e_star"]
    tc = 3.21807 * (3 * m / (4 * Es * np.sqrt(1e-3))) ** 0.4
    g = dem.system_from_scene(w.c2_wall(v0=1.0, h=tc / 200))
    g.dem_step(1200)
    assert g.dem_get_state()["vel"][0, 2] == pytest.approx(0.5, abs=1e-3)


def test_gpu_free_fall(dem):
    t = w.ds_template(6)
    scene = w.Scene(materials=np.array([w.M0]), templates=[t], planes=[], h=1e-6, gravity=np.array([0, 0, -9.81]),
                    domain_lo=np.full(3, -1.0), domain_hi=np.full(3, 1.0), gid=np.array([3], np.int64),
                    tid=np.array([0], np.int32), pos=np.zeros((1, 3)), quat=np.array([[1.0, 0, 0, 0]]),
                    vel=np.zeros((1, 3)), omega=np.zeros((1, 3)))
    g = dem.system_from_scene(scene)
    g.dem_step(1000)
    st = g.dem_get_state()
    assert st["vel"][0, 2] == pytest.approx(-1000 * 1e-6 * 9.81, rel=1e-12)
    assert st["pos"][0, 2] == pytest.approx(-4.909905e-6, rel=1e-6)


def test_gpu_momentum_conservation_zero_g(dem):
    """Mirror-exact directed rows: total momentum is conserved to round-off of the clump sums."""
    scene = w.random_clumps(46, 400, box=0.022, walls=False)
    scene.gravity[:] = 0
    g = dem.system_from_scene(scene)
    mass = np.array([t.mass for t in scene.templates])[scene.tid]
    P0 = (mass[:, None] * scene.vel).sum(0)
    scale = np.abs(mass[:, None] * scene.vel).sum()
    g.dem_step(50)
    st = g.dem_get_state()
    P = (mass[:, None] * st["vel"]).sum(0)
    assert np.abs(P - P0).max() <= 1e-12 * scale
    assert g.dem_get_stats()["n_contacts"] > 100


def test_determinism_bitwise(dem):
    scene = w.random_clumps(47, 500, box=0.03)
    a = dem.system_from_scene(scene, record_contacts=True)
    b = dem.system_from_scene(scene, record_contacts=True)
    a.dem_step(60)
    b.dem_step(60)
    sa, sb = a.dem_get_state(), b.dem_get_state()
    for k in sa:
        assert np.array_equal(sa[k], sb[k]), k
    ca, cb = a.dem_get_contacts(), b.dem_get_contacts()
    for k in ca:
        assert np.array_equal(ca[k], cb[k]), k


def test_checkpoint_resume_bitwise(dem):
    """dem_get_state + dem_get_contacts(u_t) -> dem_set_state + dem_set_contact_history resumes bitwise."""
    scene = w.random_clumps(48, 400, box=0.03)
    ref = dem.system_from_scene(scene)
    ref.dem_step(80)
    a = dem.system_from_scene(scene)
    a.dem_step(40)
    st = a.dem_get_state()
    c = a.dem_get_contacts(full=False)
    b = dem.system_from_scene(scene)
    b.dem_set_state(st["gid"], st["tid"], st["pos"], st["quat"], st["vel"], st["omega"])
    b.dem_set_contact_history(c["key_a"], c["key_b"], c["u_t"])
    b.dem_step(40)
    sr, sb = ref.dem_get_state(), b.dem_get_state()
    for k in ("pos", "quat", "vel", "omega"):
        assert np.array_equal(sr[k], sb[k]), k


def test_empty_and_lone_clump(dem):
    scene = w.c1_box()
    empty = scene.subset(np.array([], dtype=int))
    g = dem.system_from_scene(empty, record_contacts=True)
    g.dem_step(5)
    assert g.dem_get_contacts()["key_a"].size == 0
    one = scene.subset(np.array([500]))
    one.planes = []
    g = dem.system_from_scene(one, record_contacts=True)
    g.dem_step(10)
    assert g.dem_get_contacts()["key_a"].size == 0
    assert g.dem_get_stats()["steps"] == 10


def test_out_of_domain_is_reported(dem):
    scene = w.c1_box(n_side=2)
    scene.planes = []
    scene.vel[:] = 0
    scene.vel[1] = (0.0, 0.0, 1e4)  # leaves the 2 mm padded domain within a few steps
    g = dem.system_from_scene(scene)
    with pytest.raises(dem.DemError) as e:
        g.dem_step(100)
    assert e.value.status == -10 and "gid 1" in str(e.value)


def _two_spheres(pos_b, vel_a=(0.0, 0.0, 0.0), vel_b=(0.0, 0.0, 0.0)):
    t = w.sphere_template(1e-3)
    return w.Scene(materials=np.array([w.M0]), templates=[t], planes=[], h=1e-6, gravity=np.zeros(3),
                   domain_lo=np.full(3, -0.01), domain_hi=np.full(3, 0.01), gid=np.array([4, 9], np.int64),
                   tid=np.zeros(2, np.int32), pos=np.array([[0.0, 0.0, 0.0], pos_b]),
                   quat=np.array([[1.0, 0, 0, 0]] * 2), vel=np.array([vel_a, vel_b], float), omega=np.zeros((2, 3)))


def test_degenerate_contact_is_reported(dem):
    """Coincident centres of two spheres of different clumps: no contact normal exists;
    the step reports DEM_ERR_DEGENERATE_CONTACT (-12) naming both sphere keys, as the oracle
    reports its degenerate-contact error."""
    scene = _two_spheres((0.0, 0.0, 0.0))
    o = oracle.Oracle(scene)
    with pytest.raises(oracle.OracleError, match="degenerate|coincident"):
        o.step(1)
    g = dem.system_from_scene(scene)
    with pytest.raises(dem.DemError) as e:
        g.dem_step(3)
    assert e.value.status == -12
    assert "256" in str(e.value) and "576" in str(e.value)  # sphere keys 4*64 and 9*64
    with pytest.raises(dem.DemError):  # the error is latched: later calls report it again
        g.dem_step(1)


def test_nonfinite_wrench_in_step_is_reported(dem):
    """Finite inputs whose contact force overflows inside the step (relative speed 2e308: the
    normal damping term is inf) give DEM_ERR_NONFINITE (-11) naming the clump, as the
    oracle's non-finite-wrench error; the state is not advanced past the bad step."""
    scene = _two_spheres((1.9e-3, 0.0, 0.0), vel_a=(1e308, 0.0, 0.0), vel_b=(-1e308, 0.0, 0.0))
    o = oracle.Oracle(scene)
    with pytest.raises(oracle.OracleError, match="non-finite"):
        o.step(1)
    g = dem.system_from_scene(scene)
    with pytest.raises(dem.DemError) as e:
        g.dem_step(2)
    assert e.value.status == -11 and ("gid 4" in str(e.value) or "gid 9" in str(e.value))
    assert g.dem_get_stats()["steps"] <= 1


def test_capacity_regrow_keeps_parity(dem):
    """A very dense overlapping scene overflows the initial row capacity (8 per sphere):
    the library regrows and re-runs; results still match the oracle."""
    scene = w.random_clumps(49, 500, box=0.012, types=[5, 6])
    g, o = _pair(dem, scene, None)
    g.dem_step(1)
    o.step(1)
    assert g.dem_get_stats()["regrows"] >= 1
    cg, co = g.dem_get_contacts(), o.contacts()
    assert_same_contact_set(cg, co)
    assert_forces_close(cg, co, scene)


def test_row_width_regrow_keeps_parity(dem):
    """A margin of several radii gives some spheres more candidates than the initial 32
    slots of their candidate lists: the library widens them and re-runs the step; the
    contact set and forces still match the oracle."""
    scene = w.random_clumps(52, 300, box=0.02)
    g = dem.system_from_scene(scene, record_contacts=True, margin=4e-3)
    o = oracle.Oracle(scene, margin=4e-3)
    g.dem_step(1)
    o.step(1)
    co = o.contacts()
    keys, cnt = np.unique(np.concatenate([co["key_a"], co["key_b"][co["key_b"] < 2**62]]), return_counts=True)
    assert cnt.max() > 32
    assert g.dem_get_stats()["regrows"] >= 1
    cg = g.dem_get_contacts()
    assert_same_contact_set(cg, co)
    assert_forces_close(cg, co, scene)


@pytest.mark.parametrize("cell", [0.0, 1.5e-3, 8e-3])
def test_contact_set_independent_of_cell_size(dem, cell):
    scene = w.random_clumps(50, 400, box=0.03)
    g, o = _pair(dem, scene, None, cell_size=cell)
    g.dem_step(1)
    o.step(1)
    assert_same_contact_set(g.dem_get_contacts(), o.contacts())


def test_margin_false_positives(dem):
    """Margin > 0: gap contacts are in the set with zero force and zero history."""
    scene = w.random_clumps(51, 300, box=0.03)
    g, o = _pair(dem, scene, None, margin=2e-5)
    o = oracle.Oracle(scene, margin=2e-5)
    g.dem_step(1)
    o.step(1)
    cg, co = g.dem_get_contacts(), o.contacts()
    assert_same_contact_set(cg, co)
    assert (co["delta"] < 0).sum() > 5
    assert np.all(cg["force_b"][cg["delta"] <= 0] == 0)
