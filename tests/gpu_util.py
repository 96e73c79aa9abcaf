"""Shared helpers of the GPU parity tests (test infrastructure)."""
import numpy as np
import pytest


def need_gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1711_10128_b200 import build
    build.build()
    from paper_1711_10128_b200 import trplk
    return torch, trplk


def to_dev(torch, a, ld=None):
    """Host fp64 array -> CUDA tensor; a 2-D (n, k) array becomes a column-major block with ld rows."""
    a = np.asarray(a, np.float64)
    if a.ndim == 1:
        n = len(a)
        t = torch.zeros(ld or n, dtype=torch.float64, device="cuda")
        t[:n] = torch.from_numpy(a)
        return t
    n, k = a.shape
    t = torch.zeros((k, ld or n), dtype=torch.float64, device="cuda")
    t[:, :n] = torch.from_numpy(np.ascontiguousarray(a.T))
    return t


def normwise(y, yref):
    """||y - yref||_inf / ||yref||_inf."""
    y = np.asarray(y)
    yref = np.asarray(yref)
    d = np.max(np.abs(yref)) if yref.size else 0.0
    return float(np.max(np.abs(y - yref)) / d) if d > 0 else float(np.max(np.abs(y)))


def b_orthonormal_block(orc, n, k, B=None, seed=5):
    """Seeded random block orthonormalised by the ORACLE's CGS2 (B-inner product)."""
    rng = np.random.default_rng(seed)
    U = np.zeros((n, k), order="F")
    for c in range(k):
        w, h, beta, brk, _ = orc.cgs2(U[:, :c], rng.standard_normal(n), B)
        assert not brk
        U[:, c] = w / beta
    return U
