"""Thin ctypes binding of libdem_b200.so (include/dem.h) — argument marshalling only.

Every step of the hot path runs in the CUDA library; this module converts numpy arrays
to the C structs, hands the library PyTorch's caching allocator and current CUDA stream
(PyTorch is plumbing here: device memory and streams), and raises on error statuses.
There is no CPU fallback: importing this module on a machine without the built library,
or creating a system without a CUDA device, raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# DEM_LIB_PATH selects another build of the same library (A/B timing of kernel variants)
LIB_PATH = os.environ.get("DEM_LIB_PATH") or os.path.join(_HERE, "libdem_b200.so")

DEM_STATUS = {0: "ok", -1: "invalid argument", -2: "CUDA error", -3: "out of device memory", -4: "NCCL error",
              -5: "bad material", -6: "bad template", -10: "sphere out of domain", -11: "non-finite wrench",
              -12: "degenerate contact", -13: "v_max / margin exceeded", -14: "capacity", -15: "repartition needed"}

ALLOC_FN = C.CFUNCTYPE(C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p)
FREE_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p)


class dem_material(C.Structure):
    _fields_ = [("E", C.c_double), ("nu", C.c_double), ("mu", C.c_double), ("cor", C.c_double)]


class dem_template(C.Structure):
    _fields_ = [("n_comp", C.c_int32), ("offset", C.POINTER(C.c_double)), ("radius", C.POINTER(C.c_double)),
                ("material", C.POINTER(C.c_int32)), ("mass", C.c_double), ("inertia", C.c_double * 3)]


class dem_plane(C.Structure):
    _fields_ = [("point", C.c_double * 3), ("normal", C.c_double * 3), ("material", C.c_int32)]


class dem_params(C.Structure):
    _fields_ = [("h", C.c_double), ("gravity", C.c_double * 3), ("margin", C.c_double), ("cd_every", C.c_int32),
                ("domain_lo", C.c_double * 3), ("domain_hi", C.c_double * 3), ("cell_size", C.c_double),
                ("record_contacts", C.c_int32), ("alloc", ALLOC_FN), ("free", FREE_FN), ("alloc_ctx", C.c_void_p),
                ("entries_per_sphere", C.c_double), ("rank", C.c_int32), ("n_ranks", C.c_int32),
                ("slab_lo", C.c_double), ("slab_hi", C.c_double), ("halo", C.c_double), ("drift_max", C.c_double),
                ("transport", C.c_int32), ("nccl_id", C.c_ubyte * 128), ("overlap", C.c_int32)]


class dem_mesh(C.Structure):
    _fields_ = [("n_tri", C.c_int64), ("verts", C.POINTER(C.c_double)), ("material", C.c_int32),
                ("pos", C.c_double * 3), ("quat", C.c_double * 4), ("vel", C.c_double * 3), ("omega", C.c_double * 3)]


class dem_stats(C.Structure):
    _fields_ = [("steps", C.c_int64), ("n_clumps", C.c_int64), ("n_spheres", C.c_int64),
                ("n_owned_clumps", C.c_int64), ("n_owned_spheres", C.c_int64), ("n_ghost_clumps", C.c_int64),
                ("n_entries", C.c_int64), ("n_contacts", C.c_int64), ("n_inserts", C.c_int64), ("n_cells", C.c_int64),
                ("cell_size", C.c_double), ("regrows", C.c_int64), ("kernel_launches_per_step", C.c_int64),
                ("state_fast_resets", C.c_int64), ("migrated_clumps", C.c_int64), ("migration_bytes", C.c_int64),
                ("ghost_exchange_bytes", C.c_int64), ("bin_regrids", C.c_int64), ("reruns", C.c_int64)]


TRANSPORT_NCCL, TRANSPORT_LOOPBACK, TRANSPORT_PEER, TRANSPORT_LOOPBACK_PEER = 0, 1, 2, 3

EXPORTS = ["dem_create", "dem_set_state", "dem_set_contact_history", "dem_step", "dem_synchronize",
           "dem_get_state", "dem_get_contacts", "dem_get_stats", "dem_set_profiling", "dem_get_stage_times",
           "dem_status_string", "dem_last_error", "dem_destroy", "dem_nccl_unique_id", "dem_partition_plan",
           "dem_step_group", "dem_migrate", "dem_migrate_group", "dem_add_mesh", "dem_set_mesh_motion",
           "dem_get_mesh", "dem_peer_export", "dem_peer_import", "dem_migration_plan", "dem_set_state_local",
           "dem_set_state_local_group"]

_lib = None


def load_library(path: str = LIB_PATH):
    """Load libdem_b200.so (raises if it was not built — there is no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`")
    L = C.CDLL(path)
    P, I64, I32 = C.c_void_p, C.c_int64, C.c_int32
    L.dem_create.argtypes = [C.POINTER(dem_params), P, I32, P, I32, P, I32, P, C.POINTER(P)]
    L.dem_set_state.argtypes = [P, I64, P, P, P, P, P, P, I32]
    L.dem_set_contact_history.argtypes = [P, I64, P, P, P]
    L.dem_step.argtypes = [P, I64]
    L.dem_synchronize.argtypes = [P]
    L.dem_get_state.argtypes = [P, I64, C.POINTER(I64), P, P, P, P, P, P, I32]
    L.dem_get_contacts.argtypes = [P, I64, C.POINTER(I64), P, P, P, P, P, P, P]
    L.dem_get_stats.argtypes = [P, C.POINTER(dem_stats)]
    L.dem_set_profiling.argtypes = [P, I32]
    L.dem_get_stage_times.argtypes = [P, I32, P]
    L.dem_status_string.restype = C.c_char_p
    L.dem_status_string.argtypes = [C.c_int]
    L.dem_last_error.argtypes = [P, C.c_char_p, C.c_size_t]
    L.dem_destroy.argtypes = [P]
    L.dem_destroy.restype = None
    L.dem_nccl_unique_id.argtypes = [P]
    L.dem_partition_plan.argtypes = [I64, P, C.c_double, C.c_double, C.c_double, I32, I32, P, P]
    L.dem_step_group.argtypes = [P, I32, I64]
    L.dem_migrate.argtypes = [P, C.c_double, C.POINTER(I32)]
    L.dem_migrate_group.argtypes = [P, I32, C.c_double, C.POINTER(I32)]
    L.dem_add_mesh.argtypes = [P, C.POINTER(dem_mesh), C.POINTER(I32)]
    L.dem_set_mesh_motion.argtypes = [P, I32, P, P, P, P]
    L.dem_get_mesh.argtypes = [P, I32, P, P, P, P]
    L.dem_peer_export.argtypes = [P, I64, P, C.POINTER(I64)]
    L.dem_peer_import.argtypes = [P, P, P]
    L.dem_migration_plan.argtypes = [I64, P, P, P, C.c_double, C.c_double, I32, I32, P, I64, P, P]
    L.dem_set_state_local.argtypes = [P, I64, P, P, P, P, P, P]
    L.dem_set_state_local_group.argtypes = [P, I32, P, P, P, P, P, P, P]
    for f in EXPORTS:
        if f not in ("dem_destroy", "dem_status_string"):
            getattr(L, f).restype = C.c_int
    _lib = L
    return L


class DemError(RuntimeError):
    def __init__(self, status, msg=""):
        super().__init__(f"{DEM_STATUS.get(status, status)} ({status}): {msg}")
        self.status = status


def _ptr(a):
    return C.c_void_p(a.ctypes.data) if a is not None and a.size else None


def _f64(a, shape=None):
    a = np.ascontiguousarray(a, dtype=np.float64)
    return a if shape is None else a.reshape(shape)


STAGES = ["pose+bin_count", "bin_scan", "bin_scatter", "pairs", "row_scan", "rows_finish",
          "force+integrate", "halo"]


class System:
    """One dem_system on the current CUDA device and PyTorch's current stream."""

    def __init__(self, materials, templates, planes=(), *, h, gravity=(0.0, 0.0, -9.81), domain_lo, domain_hi,
                 margin=0.0, cell_size=0.0, record_contacts=False, use_torch_allocator=True, stream=None,
                 entries_per_sphere=0.0, dist=None, cd_every=1, overlap=False):
        """dist (optional): dict(rank, n_ranks, slab_lo, slab_hi, halo, drift_max, transport, nccl_id) —
        the slab decomposition of dem_params (include/dem.h); nccl_id from nccl_unique_id() on rank 0."""
        import torch  # plumbing only: device memory and streams

        if not torch.cuda.is_available():
            raise DemError(-2, "no CUDA device: the DEM hot path runs only on the GPU")
        L = load_library()
        self._torch = torch
        self.device = torch.cuda.current_device()
        self.stream = stream if stream is not None else torch.cuda.current_stream()
        mats = (dem_material * len(materials))(*[dem_material(*map(float, m)) for m in materials])
        self._keep = []
        tpls = (dem_template * len(templates))()
        for k, t in enumerate(templates):
            off, rad, mat = _f64(t["offsets"]).reshape(-1), _f64(t["radius"]), np.ascontiguousarray(t["material"],
                                                                                                    np.int32)
            self._keep += [off, rad, mat]
            tpls[k].n_comp = rad.shape[0]
            tpls[k].offset = off.ctypes.data_as(C.POINTER(C.c_double))
            tpls[k].radius = rad.ctypes.data_as(C.POINTER(C.c_double))
            tpls[k].material = mat.ctypes.data_as(C.POINTER(C.c_int32))
            tpls[k].mass = float(t["mass"])
            tpls[k].inertia[:] = [float(x) for x in t["inertia"]]
        pls = (dem_plane * max(1, len(planes)))()
        for k, (pt, nrm, m) in enumerate(planes):
            pls[k].point[:] = [float(x) for x in pt]
            pls[k].normal[:] = [float(x) for x in nrm]
            pls[k].material = int(m)
        p = dem_params()
        p.h = h
        p.gravity[:] = [float(x) for x in gravity]
        p.margin = margin
        p.cd_every = int(cd_every)
        p.overlap = 1 if overlap else 0  # next window's set detected on a second stream
        p.domain_lo[:] = [float(x) for x in domain_lo]
        p.domain_hi[:] = [float(x) for x in domain_hi]
        p.cell_size = cell_size
        p.record_contacts = 1 if record_contacts else 0
        p.entries_per_sphere = float(entries_per_sphere)
        if dist:
            p.rank, p.n_ranks = int(dist["rank"]), int(dist["n_ranks"])
            p.slab_lo, p.slab_hi = float(dist["slab_lo"]), float(dist["slab_hi"])
            p.halo, p.drift_max = float(dist["halo"]), float(dist.get("drift_max", 0.0))
            p.transport = int(dist.get("transport", TRANSPORT_NCCL))
            if dist.get("nccl_id") is not None:
                p.nccl_id[:] = list(dist["nccl_id"])
        if use_torch_allocator:
            dev = self.device

            def _alloc(nbytes, ctx, stream):
                return torch.cuda.caching_allocator_alloc(int(nbytes), dev, stream or 0)

            def _free(ptr, nbytes, ctx, stream):
                torch.cuda.caching_allocator_delete(ptr)

            self._alloc_cb, self._free_cb = ALLOC_FN(_alloc), FREE_FN(_free)
            p.alloc, p.free = self._alloc_cb, self._free_cb
        self.record = record_contacts
        self.params = p  # (read back by callers: slab bounds of a distributed rank)
        self.sys = C.c_void_p()
        rc = L.dem_create(C.byref(p), mats, len(materials), tpls, len(templates), pls, len(planes),
                          C.c_void_p(self.stream.cuda_stream), C.byref(self.sys))
        if rc:
            raise DemError(rc, "dem_create")
        self.n = 0

    # ------------------------------------------------------------------ plumbing
    def _check(self, rc, what=""):
        if rc:
            buf = C.create_string_buffer(512)
            load_library().dem_last_error(self.sys, buf, 512)
            raise DemError(rc, f"{what}: {buf.value.decode()}")

    def close(self):
        if getattr(self, "sys", None):
            load_library().dem_destroy(self.sys)
            self.sys = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ------------------------------------------------------------------ C-ABI calls
    def dem_set_state(self, gid, tid, pos, quat, vel, omega):
        """Host numpy arrays (row-major).  For device tensors use `dem_set_state_device`."""
        gid = np.ascontiguousarray(gid, np.int64)
        tid = np.ascontiguousarray(tid, np.int32)
        arr = [_f64(pos), _f64(quat), _f64(vel), _f64(omega)]
        self.n = gid.shape[0]
        self._check(load_library().dem_set_state(self.sys, self.n, _ptr(gid), _ptr(tid), *[_ptr(a) for a in arr], 0),
                    "dem_set_state")

    def dem_set_state_local(self, gid, tid, pos, quat, vel, omega):
        """Distributed, collective (NCCL ranks): rank-local input — the clumps whose COM lies in this
        rank's slab are kept (give each clump to its owner), the ghost bands come from the neighbours."""
        gid = np.ascontiguousarray(gid, np.int64)
        tid = np.ascontiguousarray(tid, np.int32)
        arr = [_f64(pos), _f64(quat), _f64(vel), _f64(omega)]
        fast0 = self.dem_get_stats()["state_fast_resets"]
        self._check(load_library().dem_set_state_local(self.sys, gid.shape[0], _ptr(gid), _ptr(tid),
                                                       *[_ptr(a) for a in arr]), "dem_set_state_local")
        # a re-layout (not the same-clumps fast path) replaced the IPC-exported arrays: re-link
        if getattr(self, "_peer", None) and self.dem_get_stats()["state_fast_resets"] == fast0:
            self.dem_peer_link(*self._peer)

    def dem_set_state_device(self, gid, tid, pos, quat, vel, omega):
        """torch CUDA tensors (int64, int32, float64 x4), contiguous."""
        ts = [gid, tid, pos, quat, vel, omega]
        self.n = gid.shape[0]
        self._check(load_library().dem_set_state(self.sys, self.n, *[C.c_void_p(t.data_ptr()) for t in ts], 1),
                    "dem_set_state")

    def dem_set_contact_history(self, key_a, key_b, u_t):
        ka, kb = np.ascontiguousarray(key_a, np.int64), np.ascontiguousarray(key_b, np.int64)
        ut = _f64(u_t)
        self._check(load_library().dem_set_contact_history(self.sys, ka.shape[0], _ptr(ka), _ptr(kb), _ptr(ut)),
                    "dem_set_contact_history")

    def dem_step(self, n_steps=1):
        self._check(load_library().dem_step(self.sys, int(n_steps)), "dem_step")

    def dem_synchronize(self):
        self._check(load_library().dem_synchronize(self.sys), "dem_synchronize")

    def dem_add_mesh(self, verts, material=0, pos=(0.0, 0.0, 0.0), quat=(1.0, 0.0, 0.0, 0.0), vel=(0.0, 0.0, 0.0),
                     omega=(0.0, 0.0, 0.0)) -> int:
        """Add a kinematic triangle mesh (verts (n_tri, 3, 3) body frame); returns its index."""
        v = _f64(verts).reshape(-1)
        m = dem_mesh()
        m.n_tri = v.shape[0] // 9
        m.verts = v.ctypes.data_as(C.POINTER(C.c_double))
        m.material = int(material)
        m.pos[:], m.quat[:], m.vel[:], m.omega[:] = [[float(x) for x in a] for a in (pos, quat, vel, omega)]
        out = C.c_int32(-1)
        self._check(load_library().dem_add_mesh(self.sys, C.byref(m), C.byref(out)), "dem_add_mesh")
        return out.value

    def dem_set_mesh_motion(self, mesh, pos, quat, vel, omega):
        arr = [_f64(x) for x in (pos, quat, vel, omega)]
        self._check(load_library().dem_set_mesh_motion(self.sys, int(mesh), *[_ptr(x) for x in arr]),
                    "dem_set_mesh_motion")

    def dem_get_mesh(self, mesh=0):
        """Pose after the last step and the wrench on the mesh from that step's contacts."""
        X, q, f, t = np.zeros(3), np.zeros(4), np.zeros(3), np.zeros(3)
        self._check(load_library().dem_get_mesh(self.sys, int(mesh), *[_ptr(x) for x in (X, q, f, t)]),
                    "dem_get_mesh")
        return dict(pos=X, quat=q, force=f, torque=t)

    def dem_peer_link(self, rank, world, group=None):
        """PEER transport: exchange the IPC export packets with the neighbouring ranks over
        torch.distributed (any backend) and map them (dem_peer_export / dem_peer_import).  Collective;
        needed after every dem_set_state (dem_migrate re-links by itself)."""
        import torch.distributed as dist

        L = load_library()
        n = C.c_int64()
        self._check(L.dem_peer_export(self.sys, 0, None, C.byref(n)), "dem_peer_export")
        buf = (C.c_ubyte * n.value)()
        self._check(L.dem_peer_export(self.sys, n.value, buf, C.byref(n)), "dem_peer_export")
        packets = [None] * world
        dist.all_gather_object(packets, bytes(buf), group=group)
        keep = [C.create_string_buffer(packets[r], len(packets[r])) if 0 <= r < world else None
                for r in (rank - 1, rank + 1)]
        self._check(L.dem_peer_import(self.sys, *[C.cast(k, C.c_void_p) if k is not None else None for k in keep]),
                    "dem_peer_import")
        self._peer = (rank, world, group)

    def dem_migrate(self, threshold=0.0) -> bool:
        """Collective (NCCL ranks): migrate clumps between slabs if an owned COM moved more than
        `threshold` [m] since the last partition (0 forces it).  True if a migration happened."""
        moved = C.c_int32(0)
        self._check(load_library().dem_migrate(self.sys, float(threshold), C.byref(moved)), "dem_migrate")
        if moved.value and getattr(self, "_peer", None):
            self.dem_peer_link(*self._peer)
        return bool(moved.value)

    def dem_get_state(self, out=None):
        """Host numpy arrays in the caller's order.  `out` (optional): preallocated arrays (e.g. in
        pinned memory) with keys gid, tid, pos, quat, vel, omega, filled in place."""
        cnt = C.c_int64()
        self._check(load_library().dem_get_state(self.sys, 0, C.byref(cnt), None, None, None, None, None, None, 0),
                    "dem_get_state")
        n = cnt.value  # owned clumps (all of them on a single system)
        if out is None:
            out = dict(gid=np.zeros(n, np.int64), tid=np.zeros(n, np.int32), pos=np.zeros((n, 3)),
                       quat=np.zeros((n, 4)), vel=np.zeros((n, 3)), omega=np.zeros((n, 3)))
        nn = C.c_int64()
        self._check(load_library().dem_get_state(self.sys, n, C.byref(nn), *[_ptr(out[k]) for k in
                                                                            ("gid", "tid", "pos", "quat", "vel",
                                                                             "omega")], 0), "dem_get_state")
        return out

    def dem_get_state_device(self, out):
        """Copy into torch CUDA tensors: dict with gid, tid, pos, quat, vel, omega."""
        nn = C.c_int64()
        ks = ("gid", "tid", "pos", "quat", "vel", "omega")
        self._check(load_library().dem_get_state(self.sys, self.n, C.byref(nn),
                                                 *[C.c_void_p(out[k].data_ptr()) for k in ks], 1), "dem_get_state")
        return out

    def dem_get_contacts(self, full=None):
        full = self.record if full is None else full
        L = load_library()
        nn = C.c_int64()
        self._check(L.dem_get_contacts(self.sys, 0, C.byref(nn), None, None, None, None, None, None, None),
                    "dem_get_contacts")
        m = nn.value
        out = dict(key_a=np.zeros(m, np.int64), key_b=np.zeros(m, np.int64), u_t=np.zeros((m, 3)))
        if full:
            out.update(force_b=np.zeros((m, 3)), point=np.zeros((m, 3)), normal=np.zeros((m, 3)), delta=np.zeros(m))
        g = lambda k: _ptr(out[k]) if k in out else None  # noqa: E731
        if m:
            self._check(L.dem_get_contacts(self.sys, m, C.byref(nn), g("key_a"), g("key_b"), g("force_b"),
                                           g("point"), g("normal"), g("u_t"), g("delta")), "dem_get_contacts")
        return out

    def dem_get_stats(self):
        st = dem_stats()
        self._check(load_library().dem_get_stats(self.sys, C.byref(st)), "dem_get_stats")
        return {k: getattr(st, k) for k, _ in dem_stats._fields_}

    def dem_set_profiling(self, enable=True):
        self._check(load_library().dem_set_profiling(self.sys, 1 if enable else 0), "dem_set_profiling")

    def dem_get_stage_times(self):
        ms = np.zeros(len(STAGES))
        self._check(load_library().dem_get_stage_times(self.sys, len(STAGES), _ptr(ms)), "dem_get_stage_times")
        return dict(zip(STAGES, ms.tolist()))


def system_from_scene(scene, record_contacts=False, cell_size=None, margin=None, local=False, **kw) -> System:
    """Build a System from a workloads.Scene-like object (duck-typed; no import of workloads).
    local=True (distributed ranks with an NCCL communicator): hand the rank only the clumps of its
    own slab (dem_set_state_local, collective); the ghost bands come from the neighbours."""
    templates = [dict(offsets=t.offsets, radius=t.radius, material=t.material, mass=t.mass, inertia=t.inertia)
                 for t in scene.templates]
    planes = [(p.point, p.normal, p.material) for p in scene.planes]
    s = System(scene.materials, templates, planes, h=scene.h, gravity=scene.gravity, domain_lo=scene.domain_lo,
               domain_hi=scene.domain_hi, margin=scene.margin if margin is None else margin,
               cell_size=scene.cell_size if cell_size is None else cell_size, record_contacts=record_contacts, **kw)
    for m in getattr(scene, "meshes", []):  # kinematic triangle meshes (NEXT-3)
        s.dem_add_mesh(m.verts, m.material, m.pos, m.quat, m.vel, m.omega)
    if local and kw.get("dist"):
        x = scene.pos[:, 0]
        sel = np.nonzero((x >= s.params.slab_lo) & (x < s.params.slab_hi))[0]
        s.dem_set_state_local(scene.gid[sel], scene.tid[sel], scene.pos[sel], scene.quat[sel], scene.vel[sel],
                              scene.omega[sel])
    else:
        s.dem_set_state(scene.gid, scene.tid, scene.pos, scene.quat, scene.vel, scene.omega)
    return s


# ---------------------------------------------------------------- distribution
def nccl_unique_id() -> bytes:
    """128-byte NCCL unique id (rank 0 creates it; the caller broadcasts it)."""
    buf = (C.c_ubyte * 128)()
    rc = load_library().dem_nccl_unique_id(C.cast(buf, C.c_void_p))
    if rc:
        raise DemError(rc, "dem_nccl_unique_id")
    return bytes(buf)


def partition_plan(pos, slab_lo, slab_hi, halo, has_left, has_right):
    """Host-only slab plan of include/dem.h: (role, send) int8 arrays per clump."""
    pos = _f64(pos).reshape(-1, 3)
    n = pos.shape[0]
    role, send = np.zeros(n, np.int8), np.zeros(n, np.int8)
    rc = load_library().dem_partition_plan(n, _ptr(pos), float(slab_lo), float(slab_hi), float(halo),
                                           int(bool(has_left)), int(bool(has_right)), _ptr(role), _ptr(send))
    if rc:
        raise DemError(rc, "dem_partition_plan")
    return role, send


def slab_bounds(x, n_ranks, lo, hi):
    """Slab faces along x with equal clump counts (rank 0 / rank n-1 extend to the domain ends)."""
    xs = np.sort(np.asarray(x))
    b = [float(lo) - 1.0]
    for r in range(1, n_ranks):
        b.append(float(xs[int(round(r * len(xs) / n_ranks))]))
    b.append(float(hi) + 1.0)
    return b


def step_group(systems, n_steps=1):
    """Lockstep a loopback-transport group (ranks 0..n-1, same GPU and stream)."""
    arr = (C.c_void_p * len(systems))(*[s.sys for s in systems])
    rc = load_library().dem_step_group(arr, len(systems), int(n_steps))
    if rc:
        buf = C.create_string_buffer(512)
        for s in systems:
            load_library().dem_last_error(s.sys, buf, 512)
            if buf.value:
                break
        raise DemError(rc, f"dem_step_group: {buf.value.decode()}")


def halo_width(scene, drift_max, margin=None):
    """Ghost band: 2 x the largest bounding radius + margin + 2 drift_max (include/dem.h); margin
    defaults to the scene's (pass the system's own if it was overridden)."""
    rb = max(float(np.max(np.linalg.norm(t.offsets, axis=1) + t.radius)) for t in scene.templates)
    return 2.0 * rb + float(scene.margin if margin is None else margin) + 2.0 * drift_max


def migrate_group(systems, threshold=0.0) -> bool:
    """dem_migrate_group: re-partition a loopback group if an owned COM moved more than
    `threshold` since the last partition (0 forces it).  Returns True if clumps were migrated."""
    arr = (C.c_void_p * len(systems))(*[s.sys for s in systems])
    moved = C.c_int32(0)
    rc = load_library().dem_migrate_group(arr, len(systems), float(threshold), C.byref(moved))
    if rc:
        buf = C.create_string_buffer(512)
        for s in systems:
            load_library().dem_last_error(s.sys, buf, 512)
            if buf.value:
                break
        raise DemError(rc, f"dem_migrate_group: {buf.value.decode()}")
    return bool(moved.value)


def _group_error(systems, rc, what):
    buf = C.create_string_buffer(512)
    for s in systems:
        load_library().dem_last_error(s.sys, buf, 512)
        if buf.value:
            break
    raise DemError(rc, f"{what}: {buf.value.decode()}")


def set_state_local_group(systems, parts):
    """dem_set_state_local_group: rank r of a loopback group gets parts[r] = (gid, tid, pos, quat,
    vel, omega) — only its own clumps are needed; the ghost bands come from the neighbours."""
    n = len(systems)
    keep = []
    cols = [[] for _ in range(6)]
    for part in parts:
        arrs = [np.ascontiguousarray(part[0], np.int64), np.ascontiguousarray(part[1], np.int32)] + \
               [_f64(x) for x in part[2:]]
        keep.append(arrs)
        for k, a in enumerate(arrs):
            cols[k].append(_ptr(a))
    n_in = np.array([len(a[0]) for a in keep], np.int64)
    ptrs = [(C.c_void_p * n)(*c) for c in cols]
    arr = (C.c_void_p * n)(*[s.sys for s in systems])
    rc = load_library().dem_set_state_local_group(arr, n, _ptr(n_in), *ptrs)
    if rc:
        _group_error(systems, rc, "dem_set_state_local_group")


def migration_plan(gid, pos, role, slab_lo, slab_hi, has_left, has_right, own_key=None):
    """Host-only migration plan of include/dem.h: (dest int8 per held clump, route int8 per directed
    row entry, given by the key of its own sphere)."""
    gid = np.ascontiguousarray(gid, np.int64)
    pos = _f64(pos).reshape(-1, 3)
    role = np.ascontiguousarray(role, np.int8)
    ok = np.ascontiguousarray(np.zeros(0) if own_key is None else own_key, np.int64)
    dest, route = np.zeros(len(gid), np.int8), np.zeros(len(ok), np.int8)
    rc = load_library().dem_migration_plan(len(gid), _ptr(gid), _ptr(pos), _ptr(role), float(slab_lo), float(slab_hi),
                                           int(bool(has_left)), int(bool(has_right)), _ptr(dest), len(ok), _ptr(ok),
                                           _ptr(route))
    if rc:
        raise DemError(rc, "dem_migration_plan")
    return dest, route
