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
