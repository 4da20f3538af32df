"""Build libdem_b200.so in-tree with nvcc for sm_100a (no JIT cache, no torch extension).

    python paper_2307_03445_b200/build.py                 # the product library
    python paper_2307_03445_b200/build.py -D NAME=1 -o x  # a variant (A/B timing via DEM_LIB_PATH)
"""
import argparse
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libdem_b200.so")
SOURCES = ["system.cu", "kernels_detect.cu", "kernels_force.cu", "kernels_scan.cu", "kernels_mesh.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "-Xcompiler", "-fPIC",
         "-shared", "-Xptxas", "-v", "--expt-relaxed-constexpr"]


def nccl_paths():
    """NCCL 2.28 shipped with the torch wheel (nvidia-nccl): include dir and libnccl.so.2."""
    import importlib.util

    spec = importlib.util.find_spec("nvidia.nccl")
    base = list(spec.submodule_search_locations)[0]
    return os.path.join(base, "include"), os.path.join(base, "lib", "libnccl.so.2")


def build(force: bool = False, verbose: bool = False, defines=(), out: str | None = None) -> str:
    lib = out or LIB
    srcs = [os.path.join(CSRC, s) for s in SOURCES]
    deps = srcs + [os.path.join(CSRC, "dem_device.cuh"), os.path.join(ROOT, "include", "dem.h")]
    if not force and not defines and os.path.exists(lib) and os.path.getmtime(lib) >= max(
            os.path.getmtime(d) for d in deps):
        return lib
    nccl_inc, nccl_lib = nccl_paths()
    cmd = [NVCC, *FLAGS, *[f"-D{d}" for d in defines], "-I", os.path.join(ROOT, "include"), "-I", nccl_inc, "-o",
           lib + ".tmp", *srcs, "-L" + os.path.dirname(nccl_lib), "-l:libnccl.so.2", "-Xlinker",
           "-rpath=" + os.path.dirname(nccl_lib)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed building " + lib)
    if verbose:
        sys.stderr.write(r.stderr)
    os.replace(lib + ".tmp", lib)
    return lib


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("-D", action="append", default=[], dest="defines")
    ap.add_argument("-o", dest="out", default=None)
    ap.add_argument("-q", action="store_true")
    a = ap.parse_args()
    print(build(force=True, verbose=not a.q, defines=a.defines, out=a.out))
