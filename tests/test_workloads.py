"""Input generator checks (no GPU): Table 1 templates and the DS mix."""
import math

import numpy as np
import pytest

import workloads as w


def test_table1_fractions_sum_and_sizes():
    assert w.DS_WEIGHT_PCT.sum() == 100.0
    for t, tpl in enumerate(w.ds_templates()):
        assert 2 * tpl.bounding_radius == pytest.approx(w.DS_SIZE_MM[t] * 1e-3, rel=1e-12)  # size = bounding diam.
        assert tpl.n_comp == w.DS_NCOMP[t]
        assert np.all(tpl.radius == w.DS_RADIUS_MM[t] * 1e-3)
        # every component overlaps a neighbour (connected union)
        d = np.linalg.norm(tpl.offsets[:, None] - tpl.offsets[None], axis=-1) + np.eye(tpl.n_comp) * 1e9
        assert np.all(d.min(1) < 2 * tpl.radius)
        # 120-degree symmetry: COM at the origin, in-plane inertia isotropic
        assert np.allclose(tpl.offsets.mean(0), 0, atol=1e-15)
        assert tpl.inertia[0] == tpl.inertia[1] and tpl.inertia[2] > tpl.inertia[0]


def test_spheres_per_clump_matches_paper_base_patch():
    """13,993,536 spheres / 4,571,136 clumps = 3.06128; fact 0.1-5 reading gives 3.06138."""
    f = w.ds_number_fractions()
    ratio = float((f * w.DS_NCOMP).sum())
    assert ratio == pytest.approx(13993536 / 4571136, abs=3e-4)
    counts = w.ds_type_counts(4571136)
    assert counts.sum() == 4571136
    assert abs(int((counts * w.DS_NCOMP).sum()) - 13993536) < 1500  # ~0.5 sigma binomial


def test_union_mass_of_sphere_and_coincident_union():
    """single sphere analytic mass/inertia within 1%; coincident spheres = one sphere."""
    m, com, I = w.union_mass_inertia(np.zeros((1, 3)), np.array([1.0]), 1.0)
    assert m == pytest.approx(4 * math.pi / 3, rel=1e-2)
    assert I[0, 0] == pytest.approx(0.4 * m, rel=1e-2)
    m2, _, _ = w.union_mass_inertia(np.zeros((2, 3)), np.array([1.0, 1.0]), 1.0)
    assert m2 == pytest.approx(m, rel=1e-12)


def test_weight_fractions_of_generated_batch():
    """generated mass per type within 2% of Table 1 on a >= 1e4 batch."""
    counts = w.ds_type_counts(20000)
    mass = np.array([t.mass for t in w.ds_templates()]) * counts
    frac = mass / mass.sum() * 100
    # sum-of-sphere-mass reading (O23) vs union masses: the union removes overlap, so
    # fractions are compared with a 2-point tolerance in percent-of-total terms
    assert np.allclose(frac, w.DS_WEIGHT_PCT, atol=2.0)


def test_c1_scene():
    s = w.c1_box()
    assert s.n_clumps == 1000 and s.n_spheres == 3000 and len(s.planes) == 6
    assert np.allclose(np.linalg.norm(s.quat, axis=1), 1, atol=1e-15)
    # bounding spheres disjoint (pitch 2.6 mm > 2.5 mm + jitter)
    d = np.linalg.norm(s.pos[:, None] - s.pos[None], axis=-1) + np.eye(1000)
    assert d.min() > 2.5e-3
