"""NEXT-3 on the GPU: kinematic triangle meshes (P:277 cone penetrometer, P:344 wheel).

The CUDA path (k_mesh_pose, k_mesh_pairs, the mesh branch of k_force_integrate, k_mesh_finish)
against the oracle's meshes (pinned in tests/test_oracle_mesh.py): bit-exact sorted contact
sets including sphere-triangle keys, per-contact forces within 1e-5, states after the run
within 1e-4, mesh poses bitwise, mesh wrenches to summation-order rounding.
"""
import numpy as np
import pytest

import oracle
from _parity import assert_forces_close, assert_same_contact_set, assert_states_close
from workloads import beds
from workloads.scenes import sphere_on_mesh

pytestmark = pytest.mark.gpu
I64 = np.iinfo(np.int64).max


@pytest.fixture(scope="module")
def dem():
    import torch

    assert torch.cuda.is_available()
    import paper_2307_03445_b200 as pkg

    return pkg


def _mesh_keys(c):
    kb = c["key_b"]
    return int(((kb <= I64 - 16) & (kb > I64 - 16 - (1 << 24))).sum())


def _assert_mesh_close(g, o, n_mesh):
    for m in range(n_mesh):
        mg, mo = g.dem_get_mesh(m), o.mesh(m)
        assert np.array_equal(mg["pos"], mo["pos"]) and np.array_equal(mg["quat"], mo["quat"]), m
        for k in ("force", "torque"):
            scale = np.abs(mo[k]).max() + 1e-30
            assert np.abs(mg[k] - mo[k]).max() <= 1e-9 * scale, (m, k, mg[k], mo[k])


@pytest.mark.parametrize("spin", [0.0, 300.0])
def test_cone_in_bed_matches_oracle(dem, spin):
    s = beds.patch_mesh(cone_speed=0.5, spin=spin)
    g = dem.system_from_scene(s, record_contacts=True)
    o = oracle.Oracle(s)
    for n in (1, 9, 20):
        g.dem_step(n)
        o.step(n)
        cg, co = g.dem_get_contacts(), o.contacts()
        assert_same_contact_set(cg, co)
        assert _mesh_keys(co) > 100
        assert_forces_close(cg, co, s)
        _assert_mesh_close(g, o, 2)
    assert_states_close(g.dem_get_state(), o.state(), dict(pos=s.pos, quat=s.quat))


@pytest.mark.parametrize("at", [(0.3e-3, -0.2e-3), (0.0, 0.0), (2.5e-3, 0.0), (1.25e-3, -1.25e-3)])
def test_one_contact_per_feature_matches_oracle(dem, at):
    """Sphere dropped on a face, the 6-triangle vertex, an edge and a diagonal of a mesh square:
    the same trajectory and wrench as the oracle (and so as the analytic plane)."""
    s = sphere_on_mesh(drop=2e-6, v0=(0.05, 0.0, -0.3), at=at)
    g = dem.system_from_scene(s, record_contacts=True)
    o = oracle.Oracle(s)
    for _ in range(4):
        g.dem_step(400)
        o.step(400)
        sg, so = g.dem_get_state(), o.state()
        for k in ("pos", "vel"):
            assert np.allclose(sg[k], so[k], rtol=1e-9, atol=1e-15), k
        _assert_mesh_close(g, o, 1)


@pytest.mark.parametrize("k,overlap", [(1, False), (4, False), (4, True)])
def test_mesh_with_deferred_overlapped_cadence(dem, k, overlap):
    s = beds.patch_mesh(cone_speed=0.5)
    # the cone starts 1 mm inside the bed: the first steps eject the spheres it overlaps at up to
    # ~100 m/s (a 1 mm Hertz overlap on a 0.8 mm sphere), so the margin covers 400 m/s
    margin = 2.0 * 400.0 * s.h * (2 * k - 2 if overlap else k)
    g = dem.system_from_scene(s, record_contacts=True, margin=margin, cd_every=k, overlap=overlap)
    o = oracle.Oracle(s, margin=margin, cd_every=k, overlap=overlap)
    for it in range(3):
        g.dem_step(k + 1)
        o.step(k + 1)
        cg, co = g.dem_get_contacts(), o.contacts()
        assert_same_contact_set(cg, co)
        assert_forces_close(cg, co, s)
    _assert_mesh_close(g, o, 2)


def test_moving_mesh_beyond_margin_is_reported(dem):
    s = beds.patch_mesh(cone_speed=30.0)
    g = dem.system_from_scene(s, margin=2.0 * 1.0 * s.h * 5, cd_every=5)
    with pytest.raises(dem.DemError) as e:
        g.dem_step(1)
    assert e.value.status == -13


def test_set_mesh_motion_midway(dem):
    """Co-simulation style: the caller re-poses the cone between steps."""
    s = beds.patch_mesh(cone_speed=0.0)
    g = dem.system_from_scene(s, record_contacts=True)
    o = oracle.Oracle(s)
    g.dem_step(5)
    o.step(5)
    X = np.array(s.meshes[1].pos) + np.array([0.2e-3, 0.0, -0.3e-3])
    q = np.array([np.cos(0.1), 0.0, np.sin(0.1), 0.0])
    v, w = np.array([0.0, 0.1, -0.4]), np.array([5.0, 0.0, 20.0])
    g.dem_set_mesh_motion(1, X, q, v, w)
    o.set_mesh_motion(1, X, q, v, w)
    g.dem_step(10)
    o.step(10)
    cg, co = g.dem_get_contacts(), o.contacts()
    assert_same_contact_set(cg, co)
    assert_forces_close(cg, co, s)
    _assert_mesh_close(g, o, 2)
