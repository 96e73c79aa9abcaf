"""Build libtrplk.so in-tree with nvcc for sm_100a (B200).

    python -m paper_1711_10128_b200.build [--force]

Links NCCL from the venv (the same libnccl.so.2 torch loads) with an rpath so
the library resolves it without LD_LIBRARY_PATH.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIBDIR = os.path.join(PKG, "lib")
LIB = os.environ.get("TRPLK_BUILD_OUT") or os.path.join(LIBDIR, "libtrplk.so")  # override: experiment builds
INCLUDE = os.path.join(ROOT, "include")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nccl_dirs():
    import nvidia.nccl as nc  # namespace package shipped with torch's CUDA wheels
    base = list(nc.__path__)[0]
    return os.path.join(base, "include"), os.path.join(base, "lib")


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu"))) + sorted(glob.glob(os.path.join(CSRC, "*.cuh")))


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = sources() + glob.glob(os.path.join(INCLUDE, "*.h")) + [__file__]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    """One nvcc process per translation unit (in parallel; kernels.cu dominates), then one link."""
    if not force and not needs_build():
        return LIB
    from concurrent.futures import ThreadPoolExecutor
    os.makedirs(os.path.dirname(LIB), exist_ok=True)
    inc, libd = _nccl_dirs()
    cus = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    objdir = os.path.join(os.path.dirname(LIB), "obj")
    os.makedirs(objdir, exist_ok=True)
    common = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-fopenmp",
              "-Xptxas", "-v" if verbose else "-O3", "-I", INCLUDE, "-I", CSRC, "-I", inc,
              *os.environ.get("TRPLK_BUILD_DEFS", "").split()]  # experiment builds: extra -D flags

    def compile_one(cu):
        obj = os.path.join(objdir, os.path.basename(cu) + ".o")
        return subprocess.run(common + ["-c", cu, "-o", obj], capture_output=True, text=True), obj

    with ThreadPoolExecutor(max_workers=len(cus)) as ex:
        results = list(ex.map(compile_one, cus))
    for r, _ in results:
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError("nvcc failed building libtrplk.so")
        if verbose:
            sys.stderr.write(r.stderr)
    cmd = [NVCC, *ARCH, "-shared", "-Xcompiler", "-fPIC,-fopenmp", *[o for _, o in results], "-o", LIB + ".tmp",
           "-L", libd, "-l:libnccl.so.2", "-Xlinker", f"-rpath,{libd}", "-lgomp"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed linking libtrplk.so")
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
