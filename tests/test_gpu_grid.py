"""Bin grid around the occupied box, re-laid out when spheres leave it.

The bins only change speed, never results: a cloud of clumps released from a small box into a
large domain flies out of its initial bin region; dem_step re-grids between step batches
(dem_stats.bin_regrids) and the contact set and states stay those of the oracle."""
import numpy as np
import pytest

import oracle
from _parity import assert_forces_close, assert_same_contact_set, assert_states_close
import workloads as w

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dem():
    import torch

    assert torch.cuda.is_available()
    import paper_2307_03445_b200 as pkg

    return pkg


def _cloud():
    from workloads.scenes import rsa_bed

    # 150 DS clumps placed without overlaps (RSA of bounding spheres) in a 24 mm cube
    from workloads.scenes import box_planes

    s = rsa_bed(21, 150, lo=(0.0, 0.0, 0.0), hi=(0.024, 0.024, 0.024))
    s.gravity = np.zeros(3)
    # an outward burst at 6 m/s into walls 12 mm outside the cube: the clumps leave the bin region
    # (the cube + 2 bins) within ~1.5 ms and hit the walls after ~2 ms
    d = s.pos - s.pos.mean(axis=0)
    s.vel = s.vel + 6.0 * d / np.linalg.norm(d, axis=1, keepdims=True)
    s.planes = box_planes(np.full(3, -0.012), np.full(3, 0.036), 0)
    s.domain_lo = np.full(3, -0.013)
    s.domain_hi = np.full(3, 0.037)
    return s


def test_regrid_when_spheres_leave_the_bin_region(dem):
    s = _cloud()
    g = dem.system_from_scene(s, record_contacts=True)
    o = oracle.Oracle(s)
    cells0 = g.dem_get_stats()["n_cells"]
    g.dem_step(2000)  # one batch (dem_step checks the status word every 2048 steps): re-grid after it
    o.step(2000)
    st = g.dem_get_stats()
    assert st["bin_regrids"] >= 1 and st["n_cells"] > cells0
    seen = 0
    for _ in range(16):  # the clumps bounce off the walls: compare every contact set met on the way
        g.dem_step(150)
        o.step(150)
        cg, co = g.dem_get_contacts(), o.contacts()
        assert_same_contact_set(cg, co)
        if len(co["key_a"]):
            assert_forces_close(cg, co, s)
        seen += len(co["key_a"])
    assert seen > 10
    assert_states_close(g.dem_get_state(), o.state(), dict(pos=s.pos, quat=s.quat))


def test_bin_region_is_the_occupied_box(dem):
    """A bed far below its domain ceiling gets bins only where it is (and 2 bins of slack)."""
    from workloads import beds

    s = beds.load_patch()
    tall = s.copy()
    tall.domain_hi = np.array(s.domain_hi, dtype=float) + np.array([0.0, 0.0, 0.5])
    a, b = dem.system_from_scene(s), dem.system_from_scene(tall)
    assert a.dem_get_stats()["n_cells"] == b.dem_get_stats()["n_cells"]
    a.dem_step(5)
    b.dem_step(5)
    sa, sb = a.dem_get_state(), b.dem_get_state()
    for k in ("pos", "quat", "vel", "omega"):
        assert np.array_equal(sa[k], sb[k]), k


@pytest.mark.parametrize("tiny", ["0", "1"])
def test_small_bin_pass_and_group_ranking_agree(dem, monkeypatch, tiny):
    """k_pairs tests bins of at most 8 members in one pass with the own-bin rule per pair (the
    small-bin pass, chosen where bins are sparse) or through the group ranking and row descriptors;
    both give the oracle's contact set and forces on a scene with every bin size up to the large-bin
    path (forced on and off here; by density the scene would take the small-bin pass)."""
    monkeypatch.setenv("DEM_PAIRS_TINY", tiny)
    scene = w.random_clumps(63, 1500, box=0.04, types=[0, 3, 6])
    g = dem.system_from_scene(scene, record_contacts=True)
    o = oracle.Oracle(scene)
    g.dem_step(1)
    o.step(1)
    assert_same_contact_set(g.dem_get_contacts(), o.contacts())
    assert_forces_close(g.dem_get_contacts(), o.contacts(), scene)
