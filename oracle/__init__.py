"""CPU fp64 oracle of the clump-DEM step — TEST INFRASTRUCTURE ONLY.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s cpu_baseline /
`--impl reference` legs may import this package.  The product path
(`paper_2307_03445_b200`) never imports it and shares no code with it.

`liboracle.so` is compiled from `dem_oracle.c` (plain C, -O2 -ffp-contract=off).
See dem_oracle.c for the per-function PAPER.md citations and DESIGN.md §3 for the
readings and the pins that check it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "dem_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
# tools/mutate_oracle.py points this at a deliberately broken build to show the pins catch it
_LIB_OVERRIDE = os.environ.get("DEM_ORACLE_LIB")
_lib = None

ORC_ERRORS = {-1: "invalid argument", -10: "out of domain", -11: "non-finite", -12: "degenerate contact"}


def build(force: bool = False) -> str:
    if _LIB_OVERRIDE:
        return _LIB_OVERRIDE
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < max(
            os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "dem_oracle.h"))):
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-std=c11", "-D_DEFAULT_SOURCE", "-fPIC",
                               "-shared", "-o", _LIB + ".tmp", _SRC, "-lm"])
        os.replace(_LIB + ".tmp", _LIB)
    return _LIB


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(build())
        P, I64, I32, D = C.c_void_p, C.c_int64, C.c_int32, C.c_double
        L.orc_create.restype = P
        L.orc_create.argtypes = [D, P, D, P, P, C.c_int, P, C.c_int, P, P, P, P, P, P, C.c_int, P, P, P, C.c_int]
        L.orc_destroy.argtypes = [P]
        L.orc_set_state.argtypes = [P, I64, P, P, P, P, P, P]
        L.orc_get_state.argtypes = [P, P, P, P, P]
        L.orc_set_history.argtypes = [P, I64, P, P, P]
        L.orc_step.argtypes = [P, I64]
        L.orc_set_cd_every.argtypes = [P, C.c_int]
        L.orc_set_overlap.argtypes = [P, C.c_int]
        L.orc_num_contacts.restype = I64
        L.orc_num_contacts.argtypes = [P]
        L.orc_steps_done.restype = I64
        L.orc_steps_done.argtypes = [P]
        L.orc_get_contacts.argtypes = [P, P, P, P, P, P, P, P]
        L.orc_get_wrench.argtypes = [P, P, P]
        L.orc_last_error.restype = C.c_char_p
        L.orc_last_error.argtypes = [P]
        L.orc_pair_params.argtypes = [P, P, P]
        L.orc_contact_force.argtypes = [D, D, D, D, D, D, D, D, P, P, P, P, P, P]
        L.orc_add_mesh.argtypes = [P, I64, P, C.c_int, P, P, P, P]
        L.orc_set_mesh_motion.argtypes = [P, C.c_int, P, P, P, P]
        L.orc_get_mesh.argtypes = [P, C.c_int, P, P, P, P]
        L.orc_closest_on_triangle.argtypes = [P, P, P, P, P]
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data if a is not None and a.size else None


def _f64(a, shape=None):
    a = np.ascontiguousarray(a, dtype=np.float64)
    return a.reshape(shape) if shape is not None else a


class OracleError(RuntimeError):
    pass


class Oracle:
    """One oracle system built from a `workloads.Scene`."""

    def __init__(self, scene, detect: int = -1, margin: float | None = None, cd_every: int = 1,
                 overlap: bool = False):
        L = lib()
        ncomp, offs, rad, mat, mass, inertia = scene.template_arrays()
        pts, nrm, pmat = scene.plane_arrays()
        self._keep = [_f64(scene.gravity), _f64(scene.domain_lo), _f64(scene.domain_hi),
                      _f64(scene.materials).reshape(-1), ncomp, _f64(offs), _f64(rad), mat, _f64(mass),
                      _f64(inertia), _f64(pts).reshape(-1), _f64(nrm).reshape(-1),
                      np.ascontiguousarray(pmat, np.int32)]
        k = self._keep
        self.h = scene.h
        self.sys = L.orc_create(scene.h, _p(k[0]), scene.margin if margin is None else margin, _p(k[1]),
                                _p(k[2]), len(scene.materials), _p(k[3]), len(scene.templates), _p(k[4]),
                                _p(k[5]), _p(k[6]), _p(k[7]), _p(k[8]), _p(k[9]), len(scene.planes),
                                _p(k[10]), _p(k[11]), _p(k[12]), detect)
        self.n = 0
        self.set_state(scene.gid, scene.tid, scene.pos, scene.quat, scene.vel, scene.omega)
        if cd_every != 1:
            self._check(L.orc_set_cd_every(self.sys, int(cd_every)))
        if overlap:  # next window's set detected one window ahead
            self._check(L.orc_set_overlap(self.sys, 1))
        for m in getattr(scene, "meshes", []):  # kinematic triangle meshes (NEXT-3)
            v = _f64(m.verts).reshape(-1)
            arr = [_f64(m.pos), _f64(m.quat), _f64(m.vel), _f64(m.omega)]
            self._keep += [v] + arr
            rc = L.orc_add_mesh(self.sys, v.shape[0] // 9, _p(v), int(m.material), *[_p(a) for a in arr])
            if rc < 0:
                self._check(rc)

    def __del__(self):
        if getattr(self, "sys", None):
            lib().orc_destroy(self.sys)
            self.sys = None

    def _check(self, rc):
        if rc:
            raise OracleError(f"{ORC_ERRORS.get(rc, rc)}: {lib().orc_last_error(self.sys).decode()}")

    def set_state(self, gid, tid, pos, quat, vel, omega):
        gid = np.ascontiguousarray(gid, np.int64)
        tid = np.ascontiguousarray(tid, np.int32)
        arr = [_f64(pos), _f64(quat), _f64(vel), _f64(omega)]
        self.n = gid.shape[0]
        self.gid = gid.copy()
        self._check(lib().orc_set_state(self.sys, self.n, _p(gid), _p(tid), *[_p(a) for a in arr]))

    def set_history(self, ka, kb, ut):
        ka = np.ascontiguousarray(ka, np.int64)
        kb = np.ascontiguousarray(kb, np.int64)
        ut = _f64(ut)
        self._check(lib().orc_set_history(self.sys, ka.shape[0], _p(ka), _p(kb), _p(ut)))

    def step(self, n: int = 1):
        self._check(lib().orc_step(self.sys, n))

    @property
    def steps_done(self) -> int:
        return lib().orc_steps_done(self.sys)

    def state(self):
        n = self.n
        pos, quat, vel, om = np.zeros((n, 3)), np.zeros((n, 4)), np.zeros((n, 3)), np.zeros((n, 3))
        lib().orc_get_state(self.sys, _p(pos), _p(quat), _p(vel), _p(om))
        return dict(gid=self.gid.copy(), pos=pos, quat=quat, vel=vel, omega=om)

    def contacts(self):
        m = lib().orc_num_contacts(self.sys)
        out = dict(key_a=np.zeros(m, np.int64), key_b=np.zeros(m, np.int64), force_b=np.zeros((m, 3)),
                   point=np.zeros((m, 3)), normal=np.zeros((m, 3)), u_t=np.zeros((m, 3)), delta=np.zeros(m))
        if m:
            lib().orc_get_contacts(self.sys, *[_p(out[k]) for k in
                                               ("key_a", "key_b", "force_b", "point", "normal", "u_t", "delta")])
        return out

    def set_mesh_motion(self, m, pos, quat, vel, omega):
        arr = [_f64(pos), _f64(quat), _f64(vel), _f64(omega)]
        self._check(lib().orc_set_mesh_motion(self.sys, int(m), *[_p(a) for a in arr]))

    def mesh(self, m=0):
        """Pose after the last step; force on the mesh and torque about its reference point from the
        last step's contacts."""
        X, q, f, t = np.zeros(3), np.zeros(4), np.zeros(3), np.zeros(3)
        self._check(lib().orc_get_mesh(self.sys, int(m), _p(X), _p(q), _p(f), _p(t)))
        return dict(pos=X, quat=q, force=f, torque=t)

    def wrench(self):
        f, t = np.zeros((self.n, 3)), np.zeros((self.n, 3))
        lib().orc_get_wrench(self.sys, _p(f), _p(t))
        return f, t


def pair_params(mat_a, mat_b):
    a, b, o = _f64(mat_a), _f64(mat_b), np.zeros(4)
    lib().orc_pair_params(_p(a), _p(b), _p(o))
    return dict(e_star=o[0], g_star=o[1], beta=o[2], mu=o[3])


def contact_force(e_star, g_star, beta, mu, r_bar, m_bar, h, delta, n, v_rel, ut):
    n, v, u = _f64(n), _f64(v_rel), _f64(ut)
    fn, ft, un = np.zeros(3), np.zeros(3), np.zeros(3)
    lib().orc_contact_force(e_star, g_star, beta, mu, r_bar, m_bar, h, delta, _p(n), _p(v), _p(u), _p(fn),
                            _p(ft), _p(un))
    return fn, ft, un


def closest_on_triangle(p, a, b, c):
    """(closest point, region): region 0 face, 1-3 edge ab/ac/bc, 4-6 vertex a/b/c."""
    p, a, b, c, o = _f64(p), _f64(a), _f64(b), _f64(c), np.zeros(3)
    reg = lib().orc_closest_on_triangle(_p(p), _p(a), _p(b), _p(c), _p(o))
    return o, reg
