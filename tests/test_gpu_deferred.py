"""NEXT-1 on the GPU: contact-set rebuild every k steps with a margin.

The GPU path with cd_every = k must match the oracle with the same cadence and margin, and
(with a sufficient margin) reproduce its own per-step-rebuild trajectory bitwise; a margin
too small for the motion is reported (DEM_ERR_VMAX) instead of silently missing contacts.
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

    assert torch.cuda.is_available()
    import paper_2307_03445_b200 as pkg

    return pkg


def _evolved_c1(steps=300):
    s = w.c1_box()
    o = oracle.Oracle(s, detect=1)
    o.step(steps)
    st = o.state()
    s.pos, s.quat, s.vel, s.omega = st["pos"], st["quat"], st["vel"], st["omega"]
    return s


@pytest.mark.parametrize("k", [5, 10])
def test_deferred_matches_oracle(dem, k):
    s = _evolved_c1()
    margin = 2.0 * 3.0 * s.h * k
    g = dem.system_from_scene(s, record_contacts=True, margin=margin, cd_every=k)
    o = oracle.Oracle(s, detect=1, margin=margin, cd_every=k)
    for _ in range(3):
        g.dem_step(k + 3)  # ends mid-window: the set of the last rebuild is compared
        o.step(k + 3)
        cg, co = g.dem_get_contacts(), o.contacts()
        assert_same_contact_set(cg, co)
        assert_forces_close(cg, co, s)
    assert_states_close(g.dem_get_state(), o.state(), dict(pos=s.pos, quat=s.quat))


def test_deferred_equals_per_step_bitwise(dem):
    s = _evolved_c1()
    ref = dem.system_from_scene(s)
    ref.dem_step(200)
    k = 10
    d = dem.system_from_scene(s, margin=2.0 * 3.0 * s.h * k, cd_every=k)
    d.dem_step(200)
    a, b = ref.dem_get_state(), d.dem_get_state()
    for key in ("pos", "quat", "vel", "omega"):
        assert np.array_equal(a[key], b[key]), key


def test_deferred_history_resume(dem):
    """Checkpoint mid-window and resume: the next step is a rebuild from the imported history."""
    s = _evolved_c1()
    k = 10
    margin = 2.0 * 3.0 * s.h * k
    ref = dem.system_from_scene(s, margin=margin, cd_every=k)
    ref.dem_step(40)
    a = dem.system_from_scene(s, margin=margin, cd_every=k)
    a.dem_step(20)
    st, c = a.dem_get_state(), a.dem_get_contacts(full=False)
    b = dem.system_from_scene(s, margin=margin, cd_every=k)
    b.dem_set_state(st["gid"], st["tid"], st["pos"], st["quat"], st["vel"], st["omega"])
    b.dem_set_contact_history(c["key_a"], c["key_b"], c["u_t"])
    b.dem_step(20)
    sr, sb = ref.dem_get_state(), b.dem_get_state()
    for key in ("pos", "quat", "vel", "omega"):
        assert np.array_equal(sr[key], sb[key]), key


def test_margin_violation_is_reported(dem):
    s = _evolved_c1()
    s.vel *= 50.0
    g = dem.system_from_scene(s, margin=1e-7, cd_every=20)
    with pytest.raises(dem.DemError) as e:
        g.dem_step(40)
    assert e.value.status == -13
