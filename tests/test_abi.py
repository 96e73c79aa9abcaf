"""CPU-side checks of the C-ABI boundary: the library loads and exports every
function that include/*.h declares (no compute calls without a GPU)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    names = set()
    for h in ("trplk.h", "trplk_kernels.h"):
        src = open(os.path.join(ROOT, "include", h)).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        for m in re.finditer(r"^\s*(?:const\s+)?[A-Za-z_][A-Za-z0-9_]*\s*\*?\s*(trplk_[a-z0-9_]+)\s*\(", src, re.M):
            names.add(m.group(1))
    return names


def test_headers_declare_the_boundary():
    names = _declared()
    for must in ("trplk_create", "trplk_solve", "trplk_destroy", "trplk_last_error", "trplk_k_step1",
                 "trplk_k_cgs2", "trplk_k_rotate", "trplk_k_sym_eig", "trplk_k_residual"):
        assert must in names


def test_library_exports_every_declared_symbol():
    from paper_1711_10128_b200 import build
    lib = ctypes.CDLL(build.build())
    missing = [n for n in _declared() if not hasattr(lib, n)]
    assert not missing, missing


def test_binding_names_match_abi():
    from paper_1711_10128_b200 import build
    build.build()
    from paper_1711_10128_b200 import trplk
    assert set(trplk.EXPORTED) == _declared()
    for n in trplk.EXPORTED:
        assert hasattr(trplk, n)


def test_options_defaults_via_abi():
    from paper_1711_10128_b200 import build
    build.build()
    from paper_1711_10128_b200 import trplk
    o = trplk.make_options()
    assert (o.seed, o.max_cycles, o.tol_mode, o.restart_size, o.lock_mode, o.use_graphs, o.precond) == (
        12, 5000, 0, 0, 0, 1, 0)


def test_library_links_sm100a_code():
    """The fat binary carries sm_100a SASS (checked with cuobjdump, no GPU needed)."""
    import shutil
    import subprocess
    from paper_1711_10128_b200 import build
    lib = build.build()
    cuobj = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(cuobj):
        pytest.skip("cuobjdump not available")
    out = subprocess.run([cuobj, "--list-elf", lib], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run([cuobj, "-sass", lib], capture_output=True, text=True).stdout
    assert "DMMA" in sass  # fp64 tensor-core rotation (K5)
