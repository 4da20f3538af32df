"""NEXT-2 on the GPU: overlapped detection cadence ("in the shadow"; P:148 one GPU, streams).

With overlap = 1 and cd_every = k, window w+1's contact set is detected on a second CUDA stream
from the sphere centres of window w's second step while window w's force steps run, and is
adopted at the next window start.  The oracle implements the same cadence (orc_set_overlap,
pinned in tests/test_oracle_deferred.py).  The GPU must match it contact for contact (false
positives included: they depend on which step's positions the set came from) and, with a margin
that covers the 2k - 2 steps of lag, reproduce its own per-step-rebuild trajectory bitwise.
"""
import os

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


def _fast(scale=20.0, steps=300):
    """The C1 box after 300 oracle steps, velocities scaled so that the detection lag matters."""
    s = w.c1_box()
    o = oracle.Oracle(s, detect=1)
    o.step(steps)
    st = o.state()
    s.pos, s.quat, s.vel, s.omega = st["pos"], st["quat"], st["vel"] * scale, st["omega"]
    return s, float(np.abs(s.vel).max() * np.sqrt(3.0))


def _same_state(a, b):
    for key in ("pos", "quat", "vel", "omega"):
        assert np.array_equal(a[key], b[key]), key


@pytest.mark.parametrize("k", [2, 5, 10])
def test_overlap_matches_oracle(dem, k):
    s, vmax = _fast()
    margin = 2.0 * vmax * s.h * (2 * k - 2) * 1.1
    g = dem.system_from_scene(s, record_contacts=True, margin=margin, cd_every=k, overlap=True)
    o = oracle.Oracle(s, detect=1, margin=margin, cd_every=k, overlap=True)
    for _ in range(4):
        g.dem_step(k + 1)  # ends at varying window phases, across adoptions
        o.step(k + 1)
        cg, co = g.dem_get_contacts(), o.contacts()
        assert_same_contact_set(cg, co)
        assert_forces_close(cg, co, s)
    assert_states_close(g.dem_get_state(), o.state(), dict(pos=s.pos, quat=s.quat))


def test_overlap_equals_per_step_bitwise(dem):
    s, vmax = _fast()
    k = 10
    ref = dem.system_from_scene(s)
    ref.dem_step(120)
    d = dem.system_from_scene(s, margin=2.0 * vmax * s.h * (2 * k - 2) * 1.1, cd_every=k, overlap=True)
    d.dem_step(120)
    _same_state(ref.dem_get_state(), d.dem_get_state())


def test_overlap_single_steps_and_profiling_match(dem):
    """dem_step(1) returns with the ahead detection still in flight on its stream; the profiled
    (in-line) schedule and the concurrent one give the same bits."""
    s, vmax = _fast()
    k = 5
    margin = 2.0 * vmax * s.h * (2 * k - 2) * 1.1
    a = dem.system_from_scene(s, margin=margin, cd_every=k, overlap=True)
    for _ in range(37):
        a.dem_step(1)
    b = dem.system_from_scene(s, margin=margin, cd_every=k, overlap=True)
    b.dem_set_profiling(True)
    b.dem_step(37)
    _same_state(a.dem_get_state(), b.dem_get_state())
    ca, cb = a.dem_get_contacts(full=False), b.dem_get_contacts(full=False)
    assert np.array_equal(ca["key_a"], cb["key_a"]) and np.array_equal(ca["u_t"], cb["u_t"])


def test_overlap_lag_is_detected(dem):
    """A margin sized for k steps of motion (enough without overlap) is too small for the 2k - 2
    steps of lag: the displacement check reports it instead of missing contacts."""
    s, vmax = _fast(scale=60.0)
    k = 10
    d = dem.system_from_scene(s, margin=2.0 * vmax * s.h * k * 0.6, cd_every=k, overlap=True)
    with pytest.raises(dem.DemError) as e:
        d.dem_step(60)
    assert e.value.status == -13


def test_overlap_ahead_overflow_recovers(dem, monkeypatch):
    """An ahead detection that overflows a capacity (fault-injected) turns the adoption into a
    rebuild at that step: the trajectory is unchanged (every contact with delta > 0 is in both
    sets) and the regrow is counted."""
    s, vmax = _fast()
    k = 5
    margin = 2.0 * vmax * s.h * (2 * k - 2) * 1.1
    ref = dem.system_from_scene(s)
    ref.dem_step(40)
    monkeypatch.setenv("DEM_FAULT_AHEAD_OVERFLOW", "2")
    d = dem.system_from_scene(s, margin=margin, cd_every=k, overlap=True)
    # dem_step enqueues all its steps before it learns of an abort (a fault is consumed per ahead
    # launch): steps 0-5 (fault at 1, the adoption at 5 aborts and re-runs as a rebuild), then
    # 6-39 (fault at 6, the adoption at 10 aborts)
    d.dem_step(6)
    d.dem_step(34)
    st = d.dem_get_stats()
    assert st["reruns"] == 2 and st["regrows"] == 0  # re-run as rebuilds; nothing needed to grow
    _same_state(ref.dem_get_state(), d.dem_get_state())


def test_overlap_needs_cd_every(dem):
    s, _ = _fast()
    with pytest.raises(dem.DemError):
        dem.system_from_scene(s, margin=1e-4, cd_every=1, overlap=True)


def test_overlap_after_a_capacity_regrow_of_the_first_rebuild(dem):
    """A wide margin overflows the initial candidate-row width in the first (in-line) rebuild; the
    ahead detections already queued behind it in the same dem_step must not touch the entry sets
    the re-run reads (regression: their row scan used to run on the stale counts)."""
    from workloads import beds

    s = beds.load_patch()
    k = 4
    margin = 2.0 * 12.0 * s.h * (2 * k - 2)
    ref = dem.system_from_scene(s)
    ref.dem_step(9)
    d = dem.system_from_scene(s, margin=margin, cd_every=k, overlap=True)
    d.dem_step(9)
    assert d.dem_get_stats()["regrows"] >= 1
    _same_state(ref.dem_get_state(), d.dem_get_state())
