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
from _parity import FORCE_RTOL, force_ref
from workloads import beds

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dem():
    import torch

    assert torch.cuda.is_available()
    import paper_2307_03445_b200 as pkg

    return pkg


def _sample_clumps(scene, k, seed):
    """k sampled clumps, biased to the interior and to large types (most contacts)."""
    rng = np.random.default_rng(seed)
    big = np.nonzero(scene.tid <= 2)[0]
    pick = list(rng.choice(big, size=min(k // 3, big.size), replace=False))
    pick += list(rng.choice(scene.n_clumps, size=k - len(pick), replace=False))
    return np.array(sorted(set(pick)))


def _crop_around(scene, c):
    rb = np.array([t.bounding_radius for t in scene.templates])
    reach = rb[scene.tid[c]] + rb.max() + 1e-4
    d = np.linalg.norm(scene.pos - scene.pos[c], axis=1)
    return np.nonzero(d <= reach)[0]


def _check_samples(gpu_contacts, gpu_state, scene, samples):
    n_checked = 0
    ka_all, kb_all = gpu_contacts["key_a"], gpu_contacts["key_b"]
    for c in samples:
        sub_idx = _crop_around(scene, c)
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
    samples = _sample_clumps(scene, 24, seed=7 if config == "c5" else 8)
    n = _check_samples(cg, sg, scene, samples)
    assert n > 100
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
    every force element by element, then states after 20 steps."""
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
    assert np.array_equal(cg["key_a"], co["key_a"]) and np.array_equal(cg["key_b"], co["key_b"])
    err = np.linalg.norm(cg["force_b"] - co["force_b"], axis=1)
    assert np.all(err <= FORCE_RTOL * np.linalg.norm(co["force_b"], axis=1) + FORCE_RTOL * force_ref(scene))
    assert len(co["key_a"]) > 100_000
    g.dem_step(19)
    o.step(19)
    sgs, sos = g.dem_get_state(), o.state()
    for k in ("vel", "omega"):
        assert np.linalg.norm(sgs[k] - sos[k]) <= 1e-6 * np.linalg.norm(sos[k])
    assert np.array_equal(g.dem_get_contacts()["key_a"], o.contacts()["key_a"])
