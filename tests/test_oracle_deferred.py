"""NEXT-1 on the oracle: contact-set rebuild every k steps with a margin.

With a margin that covers the relative motion over the window (2 v_max h k x safety),
every pair that touches during the window is already in the set; members that do not touch
have delta <= 0, hence zero force and u_t reset to 0 (reading R9) — exactly like an
absent key under per-step rebuild.  So the k > 1 trajectory must equal the k = 1 trajectory
(up to the sign of exact zeros, i.e. bitwise here), and a too-small margin must show up as a
missed contact.
"""
import numpy as np

import oracle
import workloads as w


def _evolved(steps=300):
    s = w.c1_box()
    o = oracle.Oracle(s, detect=1)
    o.step(steps)
    st = o.state()
    s.pos, s.quat, s.vel, s.omega = st["pos"], st["quat"], st["vel"], st["omega"]
    return s


def test_margin_formula_examples():
    """v = 1 m/s, h = 1e-6 s: k = 1 -> 2e-6 m; k = 20 -> 4e-5 m ("tens of microns")."""
    margin = lambda v, h, k, safety=1.0: safety * 2.0 * v * h * k  # noqa: E731
    assert margin(1.0, 1e-6, 1) == 2e-6
    assert abs(margin(1.0, 1e-6, 20) - 4e-5) < 1e-20


def test_deferred_rebuild_equals_per_step_rebuild():
    s = _evolved()
    ref = oracle.Oracle(s, detect=1)
    ref.step(200)
    k, vmax = 10, 3.0
    d = oracle.Oracle(s, detect=1, margin=2.0 * vmax * s.h * k, cd_every=k)
    d.step(200)
    a, b = ref.state(), d.state()
    for key in ("pos", "quat", "vel", "omega"):
        assert np.array_equal(a[key], b[key]), key
    # the deferred set holds false positives (gap contacts) with zero force and zero history
    c = d.contacts()
    gap = c["delta"] < 0
    assert gap.sum() > 0
    assert np.all(c["force_b"][gap] == 0) and np.all(c["u_t"][gap] == 0)
    live = c["delta"] > 0
    cr = ref.contacts()
    assert live.sum() == (cr["delta"] > 0).sum()


def test_too_small_margin_misses_contacts():
    s = _evolved()
    s.vel *= 20.0  # fast relative motion: new contacts appear inside a window
    ref = oracle.Oracle(s, detect=1)
    ref.step(60)
    d = oracle.Oracle(s, detect=1, margin=0.0, cd_every=30)
    d.step(60)
    assert not np.array_equal(ref.state()["vel"], d.state()["vel"])


# ---------------------------------------------------------------- NEXT-2: overlapped detection
# The set of window w+1 is detected from the sphere positions of the second step of window w
# (contact detection "in the shadow" of the dynamics), so it must stay complete over
# 2k - 2 steps of motion instead of k.

def _fast(scale=20.0):
    s = _evolved()
    s.vel *= scale  # relative motion large enough that the detection lag matters
    return s, float(np.abs(s.vel).max() * np.sqrt(3.0))


def test_overlap_equals_per_step_rebuild():
    s, vmax = _fast()
    k = 10
    ref = oracle.Oracle(s, detect=1)
    ref.step(60)
    d = oracle.Oracle(s, detect=1, margin=2.0 * vmax * s.h * (2 * k - 2), cd_every=k, overlap=True)
    d.step(60)
    a, b = ref.state(), d.state()
    for key in ("pos", "quat", "vel", "omega"):
        assert np.array_equal(a[key], b[key]), key


def test_overlap_lag_needs_the_larger_margin():
    """The margin of the sequential cadence (k steps of motion) suffices without overlap but
    not with it: the set adopted at a window start is k - 1 steps older."""
    s, vmax = _fast()
    k = 10
    ref = oracle.Oracle(s, detect=1)
    ref.step(60)
    seq = oracle.Oracle(s, detect=1, margin=2.0 * vmax * s.h * k, cd_every=k)
    seq.step(60)
    ovl = oracle.Oracle(s, detect=1, margin=2.0 * vmax * s.h * k, cd_every=k, overlap=True)
    ovl.step(60)
    assert np.array_equal(ref.state()["vel"], seq.state()["vel"])
    assert not np.array_equal(ref.state()["vel"], ovl.state()["vel"])


def test_overlap_set_is_the_snapshot_set():
    """Mid-window 1 the set in use is exactly the candidate set of the positions at the second
    step of window 0 (independent numpy brute force on the state after one step)."""
    from test_oracle_pins import _numpy_pairs

    s, vmax = _fast(5.0)
    k = 10
    margin = 2.0 * vmax * s.h * (2 * k - 2)
    d = oracle.Oracle(s, detect=1, margin=margin, cd_every=k, overlap=True)
    d.step(k + 3)
    c = d.contacts()
    got = list(zip(c["key_a"].tolist(), c["key_b"].tolist()))
    one = oracle.Oracle(s, detect=1)
    one.step(1)  # the state at the start of step 1 = the snapshot
    snap = s.copy()
    st = one.state()
    snap.pos, snap.quat = st["pos"], st["quat"]
    want = [(int(a), int(b)) for a, b in _numpy_pairs(snap, margin)]
    assert len(want) > 100 and got == want
