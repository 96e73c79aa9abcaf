"""Time the one-CTA Rayleigh-Ritz Jacobi kernel (tools/, measurement): python tools/eig_time.py
Prints ms per launch and sweeps for random symmetric T and for T with the TRPL+K structure
(diag(Theta) block + dense coupling), k = 20, 30, 48, 64."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1711_10128_b200 import build, inputs, trplk  # noqa: E402

build.build()
P = inputs.make("C1")
ctx = trplk.trplk_create(P.A)
rng = np.random.default_rng(3)
for k in (20, 30, 48, 64):
    M = rng.standard_normal((k, k))
    T1 = M + M.T
    T2 = np.diag(np.linspace(2.7, 3.0, k)) + 1e-3 * (M + M.T)
    for name, T in (("random", T1), ("near-diag", T2)):
        ms, sw = trplk.trplk_k_sym_eig_time(ctx, T, reps=50)
        th, Y = trplk.trplk_k_sym_eig(ctx, T)
        ref = np.linalg.eigvalsh(T)
        err = np.max(np.abs(th - ref)) / np.max(np.abs(ref))
        orth = np.max(np.abs(Y.T @ Y - np.eye(k)))
        res = np.max(np.abs(T @ Y - Y * th)) / np.max(np.abs(ref))
        if not os.environ.get("TRPLK_EIG_NEV"):
            assert err < 1e-13 and orth < 1e-13 and res < 1e-13, (k, name, err, orth, res)
        extra = ""
        if os.environ.get("TRPLK_EIG") == "tri":
            import ctypes
            clk = (ctypes.c_longlong * 8)()
            trplk._lib.trplk_debug_tri_clk(clk)
            extra = " phases(cyc): load %d tridiag %d bisect %d invit %d back %d" % tuple(
                clk[i + 1] - clk[i] for i in range(5))
        print(f"eig[{os.environ.get('TRPLK_EIG', '1b')}] k={k:2d} {name:9s}: {ms * 1e3:8.1f} us  {sw} sweeps  eig err {err:.1e} orth {orth:.1e} res {res:.1e}{extra}", flush=True)
ctx.close()
