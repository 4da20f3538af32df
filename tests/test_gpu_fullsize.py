"""Full-size parity: the configurations bench.py times, at BASELINE.json's sizes.

The GPU runs the whole bed in the bench's launch configuration; the oracle computes sampled
clumps one by one on a neighbourhood crop that contains every possible partner of the
sample (COM within R_bound(sample) + R_bound,max), so the sample's contacts, forces and
post-step state are exactly determined by the crop.  Inputs are the oracle-settled patch
tiled (workloads/beds.py) — no input comes from the CUDA path — and the first step is
compared (no history).  Properties that hold at any size are checked on the whole bed.
"""
import numpy as np
import pytest

import oracle
import workloads as w
from _parity import FORCE_RTOL, assert_forces_close, assert_same_contact_set, assert_states_close, force_ref
from workloads import beds

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dem():
    import torch

    assert torch.cuda.is_available()
    import paper_2307_03445_b200 as pkg

    return pkg


def _sample_clumps(scene, k, seed):
    """k sampled clumps spread over the bed: random interior clumps, large types (most contacts),
    clumps at the copy-paste tile seams (mirror-image tiles of the 30 mm patch), at the
    side walls, on the floor and at the free top surface."""
    rng = np.random.default_rng(seed)
    x, y, z = scene.pos[:, 0], scene.pos[:, 1], scene.pos[:, 2]
    patch = beds.load_patch()
    L = max(pl.point[0] for pl in patch.planes if pl.normal[0] < 0)  # mirror-image tiles, no gap
    fx, fy = np.mod(x, L), np.mod(y, L)
    lo, hi = scene.domain_lo + 1e-3, scene.domain_hi - np.array([1e-3, 1e-3, 0.05])
    pools = [
        (np.nonzero(scene.tid <= 2)[0], k // 5),  # big types
        (np.nonzero((np.minimum(fx, L - fx) < 2.5e-3) | (np.minimum(fy, L - fy) < 2.5e-3))[0], k // 5),  # seams
        (np.nonzero((x - lo[0] < 5e-3) | (hi[0] - x < 5e-3) | (y - lo[1] < 5e-3) | (hi[1] - y < 5e-3))[0], k // 8),
        (np.nonzero(z < 3e-3)[0], k // 10),  # floor
        (np.nonzero(z > np.quantile(z, 0.995))[0], k // 10),  # top surface
    ]
    pick = []
    for pool, m in pools:
        pick += list(rng.choice(pool, size=min(m, pool.size), replace=False))
    pick += list(rng.choice(scene.n_clumps, size=k - len(pick), replace=False))
    return np.array(sorted(set(pick)))


def _crop_around(scene, c, tree=None):
    rb = np.array([t.bounding_radius for t in scene.templates])
    reach = rb[scene.tid[c]] + rb.max() + 1e-4
    if tree is not None:
        return np.array(sorted(tree.query_ball_point(scene.pos[c], reach)))
    d = np.linalg.norm(scene.pos - scene.pos[c], axis=1)
    return np.nonzero(d <= reach)[0]


def _check_samples(gpu_contacts, gpu_state, scene, samples):
    from scipy.spatial import cKDTree

    tree = cKDTree(scene.pos)
    n_checked = 0
    ka_all, kb_all = gpu_contacts["key_a"], gpu_contacts["key_b"]
    for c in samples:
        sub_idx = _crop_around(scene, c, tree)
        sub = scene.subset(sub_idx)
        o = oracle.Oracle(sub, detect=1)
        o.step(1)
        co = o.contacts()
        gid = scene.gid[c]
        keys_c = np.arange(gid * 64, gid * 64 + 64)
        # oracle contacts involving the sample's spheres
        mo = np.isin(co["key_a"], keys_c) | np.isin(co["key_b"], keys_c)
        mg = np.isin(ka_all, keys_c) | np.isin(kb_all, keys_c)
        assert np.array_equal(co["key_a"][mo], ka_all[mg]) and np.array_equal(co["key_b"][mo], kb_all[mg]), c
        Fo, Fg = co["force_b"][mo], gpu_contacts["force_b"][mg]
        err = np.linalg.norm(Fg - Fo, axis=1)
        assert np.all(err <= FORCE_RTOL * np.linalg.norm(Fo, axis=1) + FORCE_RTOL * force_ref(scene)), c
        # post-step state of the sample clump
        so = o.state()
        j = int(np.nonzero(sub_idx == c)[0][0])
        for k in ("vel", "omega"):
            a, b = gpu_state[k][c], so[k][j]
            assert np.linalg.norm(a - b) <= 1e-9 * (np.linalg.norm(b) + 1e-3), (c, k)
        assert np.abs(gpu_state["pos"][c] - so["pos"][j]).max() <= 1e-15 + 1e-12 * np.abs(so["pos"][j]).max()
        n_checked += int(mo.sum())
    return n_checked


@pytest.mark.parametrize("config", ["c5", "c4"])
def test_full_size_sampled_parity(dem, config):
    scene = beds.c5_bed() if config == "c5" else beds.c4_bed()
    assert scene.n_clumps == (11_336_638 if config == "c5" else 2_000_000)
    g = dem.system_from_scene(scene, record_contacts=True)
    g.dem_step(1)
    cg = g.dem_get_contacts()
    sg = g.dem_get_state()
    samples = _sample_clumps(scene, 200, seed=7 if config == "c5" else 8)
    assert samples.size >= 190
    n = _check_samples(cg, sg, scene, samples)
    assert n > 1000
    # any-size properties on the whole bed: canonical keys sorted & unique, no intra-clump pairs,
    # the Coulomb cap, u_t orthogonal to n
    ka, kb = cg["key_a"], cg["key_b"]
    assert np.all(ka < kb)
    order_ok = (ka[1:] > ka[:-1]) | ((ka[1:] == ka[:-1]) & (kb[1:] > kb[:-1]))
    assert order_ok.all()
    sph = kb < np.iinfo(np.int64).max - 64
    assert np.all(ka[sph] // 64 != kb[sph] // 64)
    fn = (cg["force_b"] * cg["normal"]).sum(1)[:, None] * cg["normal"]
    ft = np.linalg.norm(cg["force_b"] - fn, axis=1)
    assert np.all(ft <= 0.6 * np.linalg.norm(fn, axis=1) * (1 + 1e-9) + 1e-300)
    st = g.dem_get_stats()
    assert st["n_contacts"] == ka.size
    print(config, "contacts", ka.size, "checked", n)


def test_dense_100k_full_parity(dem):
    """A dense 100k-clump crop of the settled bed (config-3 scale): the whole contact set and
    every force element by element at steps 1 and 100, states after 100 steps (north_star:
    states within 1e-4 relative after 100 steps)."""
    bed = beds.c5_bed()
    c = 0.5 * (bed.domain_lo + bed.domain_hi)
    half = 0.5 * np.sqrt(100_000 / 11_336_638 * 2.5 * 1.03)
    scene = beds.crop(bed, [c[0] - half, c[1] - half, -1], [c[0] + half, c[1] + half, 10])
    assert 80_000 < scene.n_clumps < 130_000
    g = dem.system_from_scene(scene, record_contacts=True)
    o = oracle.Oracle(scene, detect=1)
    g.dem_step(1)
    o.step(1)
    cg, co = g.dem_get_contacts(), o.contacts()
    assert_same_contact_set(cg, co)
    assert_forces_close(cg, co, scene)
    assert len(co["key_a"]) > 100_000
    g.dem_step(99)
    o.step(99)
    cg, co = g.dem_get_contacts(), o.contacts()
    assert_same_contact_set(cg, co)
    assert_forces_close(cg, co, scene)
    errs = assert_states_close(g.dem_get_state(), o.state(), dict(pos=scene.pos, quat=scene.quat))
    print("dense 100k, 100 steps:", errs)


def test_c3_falling_pile_parity(dem):
    """C3 (BASELINE config 3, workloads.beds.c3_impact: the 100k-clump column falling at 2 m/s onto
    a settled base layer): contact sets bit-exact and forces within 1e-5 at steps 0 (the first
    force evaluation), 1, 10 and 100, states within 1e-4 after 100 steps."""
    scene = beds.c3_impact()
    assert scene.n_clumps > 100_000
    g = dem.system_from_scene(scene, record_contacts=True)
    o = oracle.Oracle(scene, detect=1)
    done, n_max = 0, 0
    for upto in (1, 2, 11, 101):
        g.dem_step(upto - done)
        o.step(upto - done)
        done = upto
        cg, co = g.dem_get_contacts(), o.contacts()
        assert_same_contact_set(cg, co)
        assert_forces_close(cg, co, scene)
        n_max = max(n_max, len(co["key_a"]))
    assert n_max > 50_000  # the base layer's contacts and the impacts on it
    errs = assert_states_close(g.dem_get_state(), o.state(), dict(pos=scene.pos, quat=scene.quat))
    print("C3 impact, 100 steps:", n_max, errs)
