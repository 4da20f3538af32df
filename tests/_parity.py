"""Shared GPU-vs-oracle comparison helpers (tolerances from BASELINE.json north_star / SURVEY §8c)."""
import numpy as np

# north_star: per-contact forces within 1e-5 relative; states within 1e-4 relative after 100 steps
FORCE_RTOL = 1e-5
STATE_RTOL = 1e-4


def force_ref(scene):
    """F_ref = min clump mass x |g| (floor for grazing contacts, SURVEY §8c parity metrics)."""
    g = max(float(np.linalg.norm(scene.gravity)), 9.81)
    return min(t.mass for t in scene.templates) * g


def u_floor(scene):
    """Floor of the per-contact u_t comparison: h x v_ref, v_ref = the rms clump speed (>= 1 cm/s)."""
    v = np.asarray(scene.vel, float)
    vref = max(float(np.sqrt(np.mean(np.sum(v ** 2, axis=1)))) if v.size else 0.0, 0.01)
    return float(scene.h) * vref


def assert_same_contact_set(cg, co):
    assert np.array_equal(cg["key_a"], co["key_a"]) and np.array_equal(cg["key_b"], co["key_b"]), (
        f"contact sets differ: gpu {len(cg['key_a'])} vs oracle {len(co['key_a'])}")


def assert_forces_close(cg, co, scene, rtol=FORCE_RTOL):
    Fo, Fg = co["force_b"], cg["force_b"]
    err = np.linalg.norm(Fg - Fo, axis=1)
    bound = rtol * np.linalg.norm(Fo, axis=1) + rtol * force_ref(scene)
    bad = np.nonzero(err > bound)[0]
    assert bad.size == 0, f"{bad.size} contacts out of tolerance; worst {err[bad].max()} vs {bound[bad].min()}"
    for k in ("point", "normal", "delta"):
        a, b = cg[k], co[k]
        scale = np.abs(b).max() + 1e-30
        assert np.abs(a - b).max() <= 1e-9 * scale, k
    # u_t per contact (relative + a floor): the floor is the history one step of tangential
    # motion adds at the scene's speed scale (h v_ref), so a wrong or sign-flipped small u_t
    # fails even when the largest u_t of the scene is far bigger
    uo, ug = co["u_t"], cg["u_t"]
    uerr = np.linalg.norm(ug - uo, axis=1)
    ubound = rtol * np.linalg.norm(uo, axis=1) + rtol * u_floor(scene)
    ubad = np.nonzero(uerr > ubound)[0]
    assert ubad.size == 0, f"{ubad.size} u_t out of tolerance; worst {uerr[ubad].max()} vs {ubound[ubad].min()}"
    return float((err / (np.linalg.norm(Fo, axis=1) + force_ref(scene))).max()) if err.size else 0.0


def assert_states_close(sg, so, s0, rtol=STATE_RTOL):
    """V, Omega normwise and per clump; X, q by their increments."""
    out = {}
    for k in ("vel", "omega"):
        a, b = sg[k], so[k]
        nb = np.linalg.norm(b)
        if nb == 0:
            assert np.linalg.norm(a) == 0
            continue
        out[k] = float(np.linalg.norm(a - b) / nb)
        assert out[k] <= rtol, (k, out[k])
        rms = np.sqrt(np.mean(np.sum(b ** 2, axis=1)))
        per = np.linalg.norm(a - b, axis=1) <= rtol * (np.linalg.norm(b, axis=1) + rms)
        assert per.all(), (k, np.nonzero(~per)[0][:5])
    for k in ("pos", "quat"):
        da, db = sg[k] - s0[k], so[k] - s0[k]
        nb = np.linalg.norm(db)
        if nb == 0:
            continue
        out[k] = float(np.linalg.norm(da - db) / nb)
        assert out[k] <= rtol, (k, out[k])
    return out
