"""The switchable kernel paths, each through the same parity suite as the default path.

Each environment switch below selects another kernel for the same step of the method; the
kernel and solve parity tests (test_gpu_kernels.py, test_gpu_solve.py: oracle comparisons of
every kernel output and of whole solves' trajectories) are re-run in a subprocess with the switch
set (the switches are read once per process):
  TRPLK_K1=pipe     the software-pipelined K1 (k1_pipe.cuh) wherever it applies (DIA, B = I,
                    k <= 24) -- by default it runs only on slabs of >= 2^24 rows (C5)
  TRPLK_K1=rs       the two-tile register-stream K1 (stream_rs.cuh) everywhere, also on C5 slabs
  TRPLK_NO_COOP3=1  gated third-pass launches instead of the cooperative FINAL kernel
  TRPLK_NO_SMALL=1  the multi-kernel inner step also for n <= 8192 (C1)
  TRPLK_GRID=1      the cooperative grid-wide inner loop (inner_grid.cuh)
  TRPLK_EIG=tri     the tridiagonal RR eigensolver (eig_tri.cu) instead of one-CTA Jacobi
  TRPLK_K1=tpdots   the thread-per-row kernel for the first-pass CGS dots of the seed / +K vectors
  TRPLK_K1=lean     the thread-per-row inner-step K1 with register dot accumulators (lean_k1.cuh)
                    for k <= 24
  TRPLK_KPLUS=col   the +K columns one at a time (CGS2 + SpMV each), also for k_plus >= 3
  TRPLK_KPLUS=block the block +K kernels (block.cuh) also for k_plus <= 2
  TRPLK_FUSE=1      K3 of each inner step and the next K1 (and each +K column's FINAL and its
                    matvec) as one cooperative kernel, k_fin_step1 (fused.cuh)
  TRPLK_DIAC=0      every DIA diagonal as a value array (no constant-diagonal presence bits)
"""
import os
import subprocess
import sys

import pytest

from gpu_util import need_gpu

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))

VARIANTS = [("TRPLK_K1", "pipe"), ("TRPLK_K1", "rs"), ("TRPLK_K1", "tpdots"), ("TRPLK_K1", "lean"), ("TRPLK_NO_COOP3", "1"),
            ("TRPLK_NO_SMALL", "1"), ("TRPLK_GRID", "1"), ("TRPLK_EIG", "tri"), ("TRPLK_KPLUS", "col"), ("TRPLK_KPLUS", "block"),
            ("TRPLK_FUSE", "1"), ("TRPLK_DIAC", "0")]


@pytest.mark.parametrize("var,val", VARIANTS)
def test_variant_parity_suite(var, val):
    need_gpu()
    env = dict(os.environ, **{var: val})
    sel = "not full_slab and not widest and not block_kernels"  # the 2^24-row and q > 48 cases are default-path checks
    cmd = [sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider", "-m", "gpu", "-k", sel,
           os.path.join(HERE, "test_gpu_kernels.py"), os.path.join(HERE, "test_gpu_solve.py")]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=1200)
    tail = (r.stdout + r.stderr)[-3000:]
    assert r.returncode == 0, f"{var}={val}:\n{tail}"
    assert " passed" in r.stdout
