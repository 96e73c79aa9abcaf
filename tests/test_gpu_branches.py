"""The oracle's rare branches (tests/test_oracle_branches.py pins them against closed forms)
taken NATURALLY -- not forced by a debug switch -- by both the CUDA path and the oracle on the
same inputs: reading R3's third CGS pass, the R3/R16 breakdown test, the inner Krylov breakdown
(R16) on an invariant subspace."""
import numpy as np
import pytest
import scipy.sparse as sp
from types import SimpleNamespace

from gpu_util import need_gpu, normwise, to_dev

pytestmark = pytest.mark.gpu


def _frame(n, k, eta, seed=3):
    Q, _ = np.linalg.qr(np.random.default_rng(seed).standard_normal((n, k + 1)))
    V = Q[:, :k].copy(order="F")
    V[:, 1] = eta * Q[:, 0] + np.sqrt(1.0 - eta * eta) * Q[:, 1]
    return V, Q[:, k]


@pytest.mark.parametrize("n,k", [(3001, 6), (70000, 20)])
def test_cgs2_natural_third_pass(orc, n, k):
    """v_1^T v_2 = eta = 1e-4 (a basis orthonormal only to 1e-4) and w = v_1 + 1e-5 e: pass 2
    removes the eta-sized component left by pass 1 and keeps ~0.1 of the norm, so both sides take
    the third pass by reading R3's rule (no debug switch); the closed form of every pass is in
    tests/test_oracle_branches.py.  The device estimates the pass-2 norm by Pythagoras
    (||w'||^2 - ||h_2||^2 = gamma^2 - eta^4 here, against gamma^2 + eta^4), which decides the
    same way; after the third pass it computes the norm explicitly."""
    torch, trplk = need_gpu()
    eta, gamma = 1e-4, 1e-5
    A = sp.identity(n, format="csr") * 4.0
    ctx = trplk.trplk_create(A.tocsr(), n_global=n)
    V, e = _frame(n, k, eta)
    w0 = V[:, 0] + gamma * e
    out = torch.zeros(ctx.ld, dtype=torch.float64, device="cuda")
    h, beta, brk, passes = trplk.trplk_k_cgs2(ctx, to_dev(torch, V, ctx.ld), ctx.ld, k, to_dev(torch, w0, ctx.ld), out)
    w_o, h_o, beta_o, brk_o, passes_o = orc.cgs2(V, w0)
    assert passes == passes_o == 3 and not brk and not brk_o
    assert abs(beta - beta_o) <= 1e-10 * beta_o
    assert abs(beta - np.sqrt(gamma ** 2 + eta ** 6)) <= 1e-10 * beta
    assert normwise(out.cpu().numpy()[:n], w_o / beta_o) <= 1e-10
    assert np.all(np.abs(h - h_o) <= 1e-13)
    ctx.close()


@pytest.mark.parametrize("delta,brk_want", [(1e-17, True), (1e-12, False)])
def test_cgs2_breakdown_threshold_both_sides(orc, delta, brk_want):
    """w = U c + delta ||c|| e with orthonormal U: breakdown iff delta < 1e-14 (R3/R16), on both."""
    torch, trplk = need_gpu()
    n, k = 20000, 8
    A = sp.identity(n, format="csr") * 2.0
    ctx = trplk.trplk_create(A.tocsr(), n_global=n)
    Q, _ = np.linalg.qr(np.random.default_rng(7).standard_normal((n, k + 1)))
    U, e = np.asfortranarray(Q[:, :k]), Q[:, k]
    c = np.random.default_rng(8).standard_normal(k)
    w0 = U @ c + delta * np.linalg.norm(c) * e
    out = torch.zeros(ctx.ld, dtype=torch.float64, device="cuda")
    h, beta, brk, passes = trplk.trplk_k_cgs2(ctx, to_dev(torch, U, ctx.ld), ctx.ld, k, to_dev(torch, w0, ctx.ld), out)
    w_o, h_o, beta_o, brk_o, _ = orc.cgs2(U, w0)
    assert brk == brk_o == brk_want
    if not brk_want:
        # the surviving component is delta-sized, so both sides carry rounding errors of order
        # eps ||w|| in it: compare at that floor, not relative to beta
        nw = np.linalg.norm(w0)
        assert abs(beta - beta_o) <= 1e-14 * nw
        assert np.max(np.abs(out.cpu().numpy()[:n] * beta - w_o)) <= 1e-14 * nw
    ctx.close()


def _solve_both(orc, trplk, A, p, q, l, tol, **opt):
    n = A.shape[0]
    ctx = trplk.trplk_create(A, n_global=n)
    ev, X, rs, st = trplk.trplk_solve(ctx, p, q, l, tol, **opt)
    log = trplk.trplk_get_log(ctx, ph=p)
    Xh = X.cpu().numpy().copy()
    ctx.close()
    o = orc.solve(A, None, p=p, q=q, l=l, tol=tol, **opt)
    return SimpleNamespace(ev=ev, X=Xh, rs=rs, st=st, log=log), o


@pytest.mark.parametrize("reps", [20, 3000])
def test_inner_krylov_breakdown_invariant_subspace(orc, reps):
    """A = diag(1,2,3) (each value `reps` times): the inner Krylov space of eq 3.2 stays in the
    3-dimensional A-invariant span{x, Ax, A^2x}, so both sides end the inner loop after 2 columns
    (R16), the RR is exact, and the runs agree cycle by cycle: basis width 3, one cycle,
    theta_1 = 1, the same matvec count.  reps = 3000 takes the multi-kernel path (n > 8192)."""
    torch, trplk = need_gpu()
    A = sp.diags(np.repeat([1.0, 2.0, 3.0], reps)).tocsr()
    g, o = _solve_both(orc, trplk, A, 1, 8, 0, 1e-8)
    assert g.st["status"] == o["status"] == "OK"
    assert list(g.log["k"]) == list(o["log"]["k"]) == [3]
    assert g.st["a_matvecs"] == o["a_matvecs"] == 5
    assert abs(g.ev[0] - 1.0) <= 1e-14 and g.rs[0] <= 1e-13


def test_inner_breakdown_full_space(orc):
    """n = p^ + 1: the first inner CGS2 breaks down on both sides whatever the vector (the basis
    is all of R^n); the RR returns the exact spectrum in one cycle (LAPACK)."""
    torch, trplk = need_gpu()
    rng = np.random.default_rng(11)
    R = rng.standard_normal((6, 6))
    A = sp.csr_matrix(R + R.T + 8 * np.eye(6))
    g, o = _solve_both(orc, trplk, A, 5, 7, 0, 1e-8, lock_mode=1)
    assert g.st["status"] == o["status"] == "OK"
    assert list(g.log["k"]) == list(o["log"]["k"]) == [6]
    assert g.st["a_matvecs"] == o["a_matvecs"]
    assert np.max(np.abs(g.ev - np.linalg.eigvalsh(A.toarray())[:5])) <= 1e-13
