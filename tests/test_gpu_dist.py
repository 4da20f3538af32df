"""Slab decomposition on one GPU (loopback transport): P = 2, 3 ranks vs one system, bitwise.

Mirror-exact directed rows and canonical sums make every owned clump's state independent of
the decomposition, provided the ghost states are bitwise copies — so the gathered states and
contact lists of a P-rank run must equal the single-system run exactly.
"""
import numpy as np
import pytest

from workloads import beds

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dem():
    import torch

    assert torch.cuda.is_available()
    import paper_2307_03445_b200 as pkg

    return pkg


def _strip(seed=0):
    bed = beds.c5_bed()
    c = 0.5 * (bed.domain_lo + bed.domain_hi)
    s = beds.crop(bed, [c[0] - 0.07, c[1] - 0.025, -1], [c[0] + 0.07, c[1] + 0.025, 10])
    rng = np.random.default_rng(seed)
    s.vel = s.vel + rng.uniform(-0.05, 0.05, size=s.vel.shape)  # keep it moving
    return s


def _group(dem, scene, P, drift_max=1e-3, record=True, transport=None):
    halo = dem.halo_width(scene, drift_max)
    b = dem.slab_bounds(scene.pos[:, 0], P, scene.domain_lo[0], scene.domain_hi[0])
    systems = []
    for r in range(P):
        d = dict(rank=r, n_ranks=P, slab_lo=b[r], slab_hi=b[r + 1], halo=halo, drift_max=drift_max,
                 transport=dem.TRANSPORT_LOOPBACK if transport is None else transport)
        systems.append(dem.system_from_scene(scene, record_contacts=record, dist=d, entries_per_sphere=12))
    return systems


def _gather(systems):
    st = [s.dem_get_state() for s in systems]
    out = {k: np.concatenate([x[k] for x in st]) for k in st[0]}
    order = np.argsort(out["gid"])
    return {k: v[order] for k, v in out.items()}


def _contacts(systems):
    cs = [s.dem_get_contacts() for s in systems]
    out = {k: np.concatenate([x[k] for x in cs]) for k in cs[0]}
    order = np.lexsort((out["key_b"], out["key_a"]))
    return {k: v[order] for k, v in out.items()}


@pytest.mark.parametrize("P,peer", [(2, False), (3, False), (2, True), (3, True)])
def test_loopback_decomposition_is_bitwise_identical(dem, P, peer):
    """peer: the fused halo (the force kernel stores ghost states straight into the neighbour's
    arrays, flag handshake per step) instead of pack + copy + unpack."""
    scene = _strip()
    assert scene.n_clumps > 10_000
    ref = dem.system_from_scene(scene, record_contacts=True)
    ref.dem_step(30)
    sr = ref.dem_get_state()
    order = np.argsort(sr["gid"])
    sr = {k: v[order] for k, v in sr.items()}
    systems = _group(dem, scene, P, transport=dem.TRANSPORT_LOOPBACK_PEER if peer else None)
    stats = [s.dem_get_stats() for s in systems]
    assert sum(st["n_owned_clumps"] for st in stats) == scene.n_clumps
    assert all(st["n_ghost_clumps"] > 0 for st in stats)
    dem.step_group(systems, 30)
    sg = _gather(systems)
    assert np.array_equal(sg["gid"], sr["gid"])
    for k in ("pos", "quat", "vel", "omega"):
        assert np.array_equal(sg[k], sr[k]), k
    cr, cg = ref.dem_get_contacts(), _contacts(systems)
    for k in cr:
        assert np.array_equal(cg[k], cr[k]), k
    assert sum(s.dem_get_stats()["n_contacts"] for s in systems) == ref.dem_get_stats()["n_contacts"]


def test_drift_beyond_halo_guard_is_reported(dem):
    scene = _strip()
    scene.vel[:, 0] += 2.0  # 2 m/s: 0.1 mm drift in 50 steps exceeds a 20 um allowance
    systems = _group(dem, scene, 2, drift_max=20e-6, record=False)
    with pytest.raises(dem.DemError) as e:
        dem.step_group(systems, 50)
    assert e.value.status == -15


@pytest.mark.parametrize("peer", [False, True])
def test_migration_keeps_the_trajectory_bitwise(dem, peer):
    """Clumps streaming across the slab face are migrated to their new owner with their
    tangential history (dem_migrate_group); the gathered P = 2 trajectory stays
    bitwise equal to the single-system run and no drift guard fires."""
    scene = _strip(seed=3)
    scene.vel[:, 0] += 1.5  # 1.5 m/s along x: ~0.15 mm per 100 steps, across the face
    ref = dem.system_from_scene(scene, record_contacts=True)
    drift = 0.1e-3
    systems = _group(dem, scene, 2, drift_max=drift, transport=dem.TRANSPORT_LOOPBACK_PEER if peer else None)
    owned0 = [s.dem_get_stats()["n_owned_clumps"] for s in systems]
    moves = 0
    for _ in range(8):
        ref.dem_step(40)
        dem.step_group(systems, 40)
        moves += dem.migrate_group(systems, threshold=0.5 * drift)
    ref.dem_step(5)  # the contact lists of a step after the last migration
    dem.step_group(systems, 5)
    assert moves >= 3
    owned1 = [s.dem_get_stats()["n_owned_clumps"] for s in systems]
    assert owned1 != owned0 and sum(owned1) == scene.n_clumps
    sr = ref.dem_get_state()
    order = np.argsort(sr["gid"])
    sr = {k: v[order] for k, v in sr.items()}
    sg = _gather(systems)
    assert np.array_equal(sg["gid"], sr["gid"])
    for k in ("pos", "quat", "vel", "omega"):
        assert np.array_equal(sg[k], sr[k]), k
    cr, cg = ref.dem_get_contacts(), _contacts(systems)
    for k in ("key_a", "key_b", "u_t", "force_b"):
        assert np.array_equal(cg[k], cr[k]), k


def test_migration_below_threshold_is_a_no_op(dem):
    scene = _strip()
    systems = _group(dem, scene, 2, record=False)
    dem.step_group(systems, 5)
    owned = [s.dem_get_stats()["n_owned_clumps"] for s in systems]
    assert not dem.migrate_group(systems, threshold=1.0)
    assert [s.dem_get_stats()["n_owned_clumps"] for s in systems] == owned


@pytest.mark.parametrize("peer", [False, True])
def test_distributed_fast_reset_equals_fresh_group(dem, peer):
    """dem_set_state with the same global clumps and the same slab partition takes the fast
    path on every rank (device permutation, drift reference refreshed, step counts and peer flag
    words reset); the group then steps exactly like a freshly built one."""
    scene = _strip(seed=5)
    tr = dem.TRANSPORT_LOOPBACK_PEER if peer else None
    a = _group(dem, scene, 2, record=False, transport=tr)
    dem.step_group(a, 25)
    t = scene.copy()
    t.vel = scene.vel[::-1].copy()
    for s in a:
        s.dem_set_state(t.gid, t.tid, t.pos, t.quat, t.vel, t.omega)
        assert s.dem_get_stats()["state_fast_resets"] == 1
    b = _group(dem, t, 2, record=False, transport=tr)
    dem.step_group(a, 30)
    dem.step_group(b, 30)
    ga, gb = _gather(a), _gather(b)
    for k in ("gid", "pos", "quat", "vel", "omega"):
        assert np.array_equal(ga[k], gb[k]), k


@pytest.mark.parametrize("peer,overlap", [(False, False), (True, False), (True, True)])
def test_distributed_deferred_cadence_is_bitwise_identical(dem, peer, overlap):
    """Slab decomposition with the deferred (and overlapped) contact-set cadence: the gathered
    states equal the single-system per-step-rebuild run bitwise (every contact with delta > 0 is
    in every set; sums are canonical; ghosts are bitwise copies)."""
    scene = _strip(seed=7)
    ref = dem.system_from_scene(scene)
    ref.dem_step(40)
    k = 5
    vmax = float(np.abs(scene.vel).max() * np.sqrt(3.0)) + 1.0
    margin = 2.0 * vmax * scene.h * ((2 * k - 2) if overlap else k)
    drift = 1e-3
    halo = dem.halo_width(scene, drift) + margin
    b = dem.slab_bounds(scene.pos[:, 0], 2, scene.domain_lo[0], scene.domain_hi[0])
    systems = []
    for r in range(2):
        d = dict(rank=r, n_ranks=2, slab_lo=b[r], slab_hi=b[r + 1], halo=halo, drift_max=drift,
                 transport=dem.TRANSPORT_LOOPBACK_PEER if peer else dem.TRANSPORT_LOOPBACK)
        systems.append(dem.system_from_scene(scene, dist=d, entries_per_sphere=16, margin=margin, cd_every=k,
                                             overlap=overlap))
    dem.step_group(systems, 40)
    sr = ref.dem_get_state()
    o = np.argsort(sr["gid"])
    sg = _gather(systems)
    for key in ("gid", "pos", "quat", "vel", "omega"):
        assert np.array_equal(sg[key], sr[key][o]), key


def _owner(systems):
    return {int(g): r for r, s in enumerate(systems) for g in s.dem_get_state()["gid"]}


@pytest.mark.parametrize("peer", [False, True])
def test_migration_moves_only_the_crossers(dem, peer):
    """Neighbour-only migration: each rank sends only the clumps whose COM crossed
    into a neighbour's slab (and the contacts routed with them), so the migrated clump count equals
    the number of owner changes and the bytes moved scale with it, not with the system."""
    scene = _strip(seed=4)
    scene.vel[:, 0] += 1.5
    drift = 0.1e-3
    systems = _group(dem, scene, 3, drift_max=drift, transport=dem.TRANSPORT_LOOPBACK_PEER if peer else None)
    for _ in range(3):
        dem.step_group(systems, 40)
        before = _owner(systems)
        assert dem.migrate_group(systems, threshold=0.5 * drift)
        after = _owner(systems)
        changed = sum(1 for g in before if before[g] != after[g])
        st = [s.dem_get_stats() for s in systems]
        assert sum(x["migrated_clumps"] for x in st) == changed > 0
        # per crosser: its 15-double record plus the directed row entries of its (at most 6)
        # spheres, 5 doubles each; 2 count words per side and rank — far below the 15 doubles per
        # clump of the whole system an all-gather would move
        mb = sum(x["migration_bytes"] for x in st)
        assert mb <= 8 * (4 * len(systems) + changed * (15 + 5 * 80))
        assert mb < 0.05 * 8 * 15 * scene.n_clumps
        ghosts = sum(x["n_ghost_clumps"] for x in st)
        assert sum(x["ghost_exchange_bytes"] for x in st) == 8 * 15 * ghosts


@pytest.mark.parametrize("peer", [False, True])
def test_rank_local_set_state_equals_global_input(dem, peer):
    """dem_set_state_local_group: every rank is given only the clumps it owns (its slab); the ghost
    bands come from the neighbours.  The group then steps bitwise like one built from the global
    state on every rank."""
    scene = _strip(seed=6)
    tr = dem.TRANSPORT_LOOPBACK_PEER if peer else None
    a = _group(dem, scene, 3, record=False, transport=tr)
    b = _group(dem, scene, 3, record=False, transport=tr)
    parts = []
    for s in b:
        sel = np.nonzero((scene.pos[:, 0] >= s.params.slab_lo) & (scene.pos[:, 0] < s.params.slab_hi))[0]
        sub = scene.subset(sel)
        parts.append((sub.gid, sub.tid, sub.pos, sub.quat, sub.vel, sub.omega))
    dem.set_state_local_group(b, parts)
    sa, sb = [s.dem_get_stats() for s in a], [s.dem_get_stats() for s in b]
    for x, y in zip(sa, sb):
        assert (x["n_owned_clumps"], x["n_ghost_clumps"]) == (y["n_owned_clumps"], y["n_ghost_clumps"])
    dem.step_group(a, 30)
    dem.step_group(b, 30)
    ga, gb = _gather(a), _gather(b)
    for k in ("gid", "pos", "quat", "vel", "omega"):
        assert np.array_equal(ga[k], gb[k]), k


@pytest.mark.parametrize("peer", [False, True])
def test_coordinated_capacity_regrow(dem, peer):
    """One rank starts with far too little row capacity: its overflow aborts the step on every rank
    (the abort vote before the force kernels), each rank regrows what overflowed on it, and all
    re-run — the gathered trajectory stays bitwise equal to the single system's."""
    scene = _strip(seed=8)
    ref = dem.system_from_scene(scene)
    ref.dem_step(25)
    drift = 1e-3
    halo = dem.halo_width(scene, drift)
    b = dem.slab_bounds(scene.pos[:, 0], 2, scene.domain_lo[0], scene.domain_hi[0])
    systems = []
    for r in range(2):
        d = dict(rank=r, n_ranks=2, slab_lo=b[r], slab_hi=b[r + 1], halo=halo, drift_max=drift,
                 transport=dem.TRANSPORT_LOOPBACK_PEER if peer else dem.TRANSPORT_LOOPBACK)
        systems.append(dem.system_from_scene(scene, dist=d, entries_per_sphere=12 if r == 0 else 0.05))
    dem.step_group(systems, 25)
    st = [s.dem_get_stats() for s in systems]
    assert st[0]["regrows"] == 0 and st[1]["regrows"] >= 1
    sr = ref.dem_get_state()
    o = np.argsort(sr["gid"])
    sg = _gather(systems)
    for k in ("gid", "pos", "quat", "vel", "omega"):
        assert np.array_equal(sg[k], sr[k][o]), k
