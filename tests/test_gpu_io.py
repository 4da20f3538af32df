"""State I/O through the C-ABI (include/dem.h dem_set_state / dem_get_state).

dem_set_state with the same clumps as the previous call takes a fast path (the state is permuted
into the existing storage order on the device, no re-layout); it must be indistinguishable from
a fresh system: same bits after stepping, history cleared, caller order preserved.
"""
import numpy as np
import pytest

import workloads as w

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dem():
    import torch

    assert torch.cuda.is_available()
    import paper_2307_03445_b200 as pkg

    return pkg


def _moved(s, seed=4):
    rng = np.random.default_rng(seed)
    t = s.copy()
    t.pos = s.pos + rng.uniform(-2e-5, 2e-5, size=s.pos.shape)
    t.vel = s.vel[::-1].copy()
    return t


def test_fast_reset_equals_fresh_system(dem):
    s = w.c1_box()
    a = dem.system_from_scene(s)
    a.dem_step(120)  # leaves history and a non-zero ping-pong phase behind
    t = _moved(s)
    a.dem_set_state(t.gid, t.tid, t.pos, t.quat, t.vel, t.omega)
    assert a.dem_get_stats()["steps"] == 0 and a.dem_get_stats()["state_fast_resets"] == 1
    b = dem.system_from_scene(t)
    a.dem_step(150)
    b.dem_step(150)
    sa, sb = a.dem_get_state(), b.dem_get_state()
    for k in ("gid", "pos", "quat", "vel", "omega"):
        assert np.array_equal(sa[k], sb[k]), k
    ca, cb = a.dem_get_contacts(full=False), b.dem_get_contacts(full=False)
    assert np.array_equal(ca["key_a"], cb["key_a"]) and np.array_equal(ca["u_t"], cb["u_t"])


def test_get_state_returns_the_caller_order(dem):
    s = w.random_clumps(7, 300, box=0.03)
    g = dem.system_from_scene(s)
    st = g.dem_get_state()
    assert np.array_equal(st["gid"], s.gid) and np.array_equal(st["tid"], s.tid)
    assert np.array_equal(st["pos"], s.pos) and np.array_equal(st["quat"], s.quat)
    # a fast-path reset keeps the caller order too
    t = _moved(s)
    g.dem_set_state(t.gid, t.tid, t.pos, t.quat, t.vel, t.omega)
    st = g.dem_get_state()
    assert np.array_equal(st["pos"], t.pos) and np.array_equal(st["vel"], t.vel)


def test_fast_reset_rejects_non_finite(dem):
    s = w.c1_box()
    g = dem.system_from_scene(s)
    t = s.copy()
    t.vel = t.vel.copy()
    t.vel[17, 1] = np.nan
    with pytest.raises(dem.DemError) as e:
        g.dem_set_state(t.gid, t.tid, t.pos, t.quat, t.vel, t.omega)
    assert e.value.status == -11
