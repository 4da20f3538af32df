"""C-ABI library checks that need no GPU: it builds, loads and exports every declared symbol."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "dem.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(dem_[a-z_]+)\s*\(", src)))


def test_library_builds_and_exports_every_declared_symbol():
    from paper_2307_03445_b200 import build as b

    lib = b.build()
    out = subprocess.run(["nm", "-D", "--defined-only", lib], capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r" T (dem_\w+)", out))
    declared = _declared()
    assert len(declared) >= 12
    missing = [d for d in declared if d not in exported]
    assert not missing, missing
    import paper_2307_03445_b200 as pkg

    L = pkg.load_library()
    for d in declared:
        assert hasattr(L, d)
    assert set(pkg.EXPORTS) == set(declared)


def test_status_strings_without_gpu():
    import paper_2307_03445_b200 as pkg

    L = pkg.load_library()
    assert L.dem_status_string(0) == b"ok"
    assert L.dem_status_string(-10) == b"sphere out of domain"


def test_binding_refuses_without_cuda():
    import torch

    import paper_2307_03445_b200 as pkg
    import workloads as w

    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    with pytest.raises(pkg.DemError):
        pkg.system_from_scene(w.c1_box())


def test_sm100a_cubin_and_no_oracle_link():
    """The product is compiled for sm_100a and never links/loads the oracle."""
    from paper_2307_03445_b200 import build as b

    lib = b.build()
    out = subprocess.run(["cuobjdump", "--list-elf", lib], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    deps = subprocess.run(["ldd", lib], capture_output=True, text=True).stdout
    assert "oracle" not in deps
    for f in os.listdir(os.path.join(ROOT, "paper_2307_03445_b200")):
        if f.endswith(".py"):
            txt = open(os.path.join(ROOT, "paper_2307_03445_b200", f)).read()
            assert "import oracle" not in txt and "from oracle" not in txt


def test_dem_create_rejects_a_thin_ghost_band_without_gpu():
    """A distributed system's ghost band must be >= 2 R_bound,max + margin + 2 drift_max
    (include/dem.h): dem_create refuses a thinner one before touching the GPU."""
    import ctypes as C

    import numpy as np

    import paper_2307_03445_b200 as pkg
    from paper_2307_03445_b200 import binding as B

    L = pkg.load_library()
    mats = (B.dem_material * 1)(B.dem_material(1e9, 0.3, 0.4, 0.5))
    off, rad, mat = np.array([0.0, 0.0, 0.0, 1e-3, 0.0, 0.0]), np.array([1e-3, 1e-3]), np.zeros(2, np.int32)
    tp = (B.dem_template * 1)()
    tp[0].n_comp = 2
    tp[0].offset = off.ctypes.data_as(C.POINTER(C.c_double))
    tp[0].radius = rad.ctypes.data_as(C.POINTER(C.c_double))
    tp[0].material = mat.ctypes.data_as(C.POINTER(C.c_int32))
    tp[0].mass = 1e-5
    tp[0].inertia[:] = [1e-11, 1e-11, 1e-11]
    p = B.dem_params()
    p.h = 1e-6
    p.gravity[:] = [0, 0, -9.81]
    p.cd_every = 2
    p.margin = 1e-5
    p.domain_lo[:] = [-1, -1, -1]
    p.domain_hi[:] = [1, 1, 1]
    p.rank, p.n_ranks, p.slab_lo, p.slab_hi, p.drift_max = 0, 2, -1.0, 0.0, 1e-4
    p.transport = B.TRANSPORT_LOOPBACK
    need = 2 * 2e-3 + 1e-5 + 2 * 1e-4  # R_bound = 2 mm
    out = C.c_void_p()
    p.halo = need * (1 - 1e-6)
    assert L.dem_create(C.byref(p), mats, 1, tp, 1, None, 0, None, C.byref(out)) == -1
    assert not out.value
