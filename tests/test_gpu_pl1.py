"""PL+1 (Algorithm 2, NEXT-1 of SURVEY 8(f)) through the C ABI against the oracle
(orc_pl1_solve, readings P1-P6): the same iteration count and A-matvec count, the per-iteration
Rayleigh quotients rho_k to 1e-10 relative, the final rho to 1e-12, the same B-normalised
iterate, and the step-7 conjugacy identity on the device."""
import numpy as np
import pytest

from gpu_util import need_gpu

pytestmark = pytest.mark.gpu


def _run(trplk, orc, P, m, tol, variant=0, use_precond=True, fmt="auto"):
    import os
    if fmt == "sell":
        os.environ["TRPLK_FORCE_SELL"] = "1"
    try:
        ctx = trplk.trplk_create(P.A, P.B, P.sigma)
    finally:
        os.environ.pop("TRPLK_FORCE_SELL", None)
    rho, res, x, st, log = trplk.trplk_pl1_solve(ctx, m, tol, variant=variant, use_precond=use_precond)
    xg = x.cpu().numpy().copy()
    ctx.close()
    o = orc.pl1_solve(P.A, P.B, m=m, tol=tol, sigma=P.sigma, variant=variant, use_precond=use_precond)
    return rho, res, xg, st, log, o


@pytest.mark.parametrize("name,N,m,variant,prec,fmt", [
    ("C2", 16, 4, 0, True, "auto"),
    ("C2", 16, 4, 0, True, "sell"),
    ("C3", 12, 1, 0, True, "auto"),     # m = 1: the LOPCG-like end of the family
    ("C2", 24, 1, 1, True, "auto"),     # m = 1, practical step 7 (the paper's stagnates here: DESIGN P4)
    ("C2", 16, 6, 1, True, "auto"),     # practical step 7
    ("C2", 12, 3, 0, False, "auto"),    # M = I
    ("C4", 8, 4, 0, True, "auto"),      # pencil, B != I
    ("C3", 12, 4, 0, True, "auto"),     # multiple lambda_2: lambda_1 simple
])
def test_pl1_parity(orc, gen, name, N, m, variant, prec, fmt):
    torch, trplk = need_gpu()
    P = gen.make(name, N=N)
    tol = 1e-9
    rho, res, x, st, log, o = _run(trplk, orc, P, m, tol, variant, prec, fmt)
    assert st["status"] == "OK" and o["status"] == "OK"
    assert st["cycles"] == o["cycles"]
    assert st["a_matvecs"] == o["a_matvecs"]
    assert res <= tol
    lo = o["log"]
    assert len(log["rho"]) == len(lo["rho"])
    assert np.max(np.abs(log["rho"] - lo["rho"]) / np.abs(lo["rho"])) <= 1e-10
    assert abs(rho - o["rho"]) <= 1e-12 * abs(o["rho"])
    B = None if P.B is None else P.B.to_scipy()
    Bx = x if B is None else B @ x
    assert abs(x @ Bx - 1) <= 1e-12
    assert abs(abs(Bx @ o["x"]) - 1) <= 1e-8
    if variant == 0:
        assert np.max(np.abs(log["conj"])) <= 1e-10


def test_pl1_full_size_C2(orc, gen):
    """BASELINE C2 size (262,144 rows), m = 4: same trajectory as the oracle."""
    torch, trplk = need_gpu()
    P = gen.make("C2")
    rho, res, x, st, log, o = _run(trplk, orc, P, 4, 1e-8)
    assert st["status"] == "OK" and o["status"] == "OK"
    assert st["cycles"] == o["cycles"] and st["a_matvecs"] == o["a_matvecs"]
    assert np.max(np.abs(log["rho"] - o["log"]["rho"]) / np.abs(o["log"]["rho"])) <= 1e-10
    assert abs(rho - o["rho"]) <= 1e-12 * abs(o["rho"])
    assert abs(abs(x @ o["x"]) - 1) <= 1e-8


def test_pl1_wide_block_and_breakdown(orc, gen):
    """m = 12 (Gram by the per-column fused dot kernel, NC = 14 > 8) on C2, and a Krylov
    breakdown: A with 4 distinct eigenvalues (n = 64), m = 6 -> G_k ends after <= 3 columns
    (step 4, P1) on the oracle and the GPU alike."""
    import scipy.sparse as sp
    torch, trplk = need_gpu()
    P = gen.make("C2", N=12)
    rho, res, x, st, log, o = _run(trplk, orc, P, 12, 1e-9)
    assert st["status"] == "OK" and o["status"] == "OK"
    assert st["cycles"] == o["cycles"] and st["a_matvecs"] == o["a_matvecs"]
    assert abs(rho - o["rho"]) <= 1e-12 * abs(o["rho"])

    class _M:  # CSR in the shape inputs.make returns
        def __init__(self, S):
            S = S.tocsr()
            self.rowptr = S.indptr.astype(np.int64)
            self.col = S.indices.astype(np.int64)
            self.val = S.data.astype(np.float64)
            self.n = S.shape[0]
            self.row_begin = 0

        def to_scipy(self):
            return sp.csr_matrix((self.val, self.col, self.rowptr), shape=(self.n, self.n))

    # x_0 in a 2-dimensional invariant subspace: v_2 = (A - rho) g_1 lies in span{x_0, g_1},
    # so CGS2 against g_1 alone returns ~x_0 (g_2), v_3 breaks down (mg = 2), and Q = [x, g_1, g_2]
    # is singular on x -> BREAKDOWN (P3) at iteration 0, oracle and GPU alike
    d = np.arange(1.0, 65.0)
    A = _M(sp.diags(d))
    x0 = np.zeros(64)
    x0[0] = x0[1] = 1.0
    ctx = trplk.trplk_create(A, None, 0.0)
    rho, res, x, st, log = trplk.trplk_pl1_solve(ctx, 6, 1e-10, use_precond=False, x0=x0)
    ctx.close()
    o = orc.pl1_solve(A, None, m=6, tol=1e-10, use_precond=False, x0=x0)
    assert o["status"] == "BREAKDOWN" and st["status"] == "BREAKDOWN"
    assert o["log"]["mg"][0] == 2
    assert st["cycles"] == o["cycles"] == 0 and st["a_matvecs"] == o["a_matvecs"]
    assert abs(rho - o["rho"]) <= 1e-14


@pytest.mark.parametrize("name,N,m", [("C2", 16, 4), ("C2", 12, 1), ("C4", 8, 2), ("C3", 10, 3)])
def test_pl1_quasi_optimality(orc, gen, name, N, m):
    """Global quasi-optimality diagnostic (reading P7, Def. defnglbopt) on the
    device against the oracle: the same dim U_k sequence, rho(y*_k) to 1e-10 relative, the ratio
    (rho_k - rho(y*_k)) / (rho_k - lambda_1) to 1e-5 where rho_k - lambda_1 > 1e-4 |lambda_1|;
    arming it leaves the PL+1 trajectory bit-identical."""
    torch, trplk = need_gpu()
    P = gen.make(name, N=N)
    tol = 1e-9
    ctx = trplk.trplk_create(P.A, P.B, P.sigma)
    rho0, _, x0, st0, log0 = trplk.trplk_pl1_solve(ctx, m, tol)
    x0 = x0.cpu().numpy().copy()
    assert trplk.trplk_pl1_get_qopt(ctx)["rho_star"].size == 0  # off by default
    trplk.trplk_pl1_set_qopt(ctx, 64)
    rho, _, x, st, log = trplk.trplk_pl1_solve(ctx, m, tol)
    q = trplk.trplk_pl1_get_qopt(ctx)
    ctx.close()
    assert rho == rho0 and np.array_equal(log["rho"], log0["rho"])
    assert np.array_equal(x.cpu().numpy(), x0)
    assert st["a_matvecs"] == st0["a_matvecs"] and st["kernel_launches"] == st0["kernel_launches"]
    o = orc.pl1_solve(P.A, P.B, m=m, tol=tol, sigma=P.sigma, qopt_cap=64)
    oq, od = o["log"]["qopt"], o["log"]["qdim"]
    assert len(q["rho_star"]) == len(oq) == min(len(log["rho"]), 64) >= 3
    assert np.array_equal(q["dim"], od)
    assert np.max(np.abs(q["rho_star"] - oq) / np.abs(oq)) <= 1e-10
    lam = o["rho"]
    orat = (o["log"]["rho"][:len(oq)] - oq) / (o["log"]["rho"][:len(oq)] - lam)
    sel = (o["log"]["rho"][:len(oq)] - lam) > 1e-4 * abs(lam)
    assert sel.sum() >= 2
    assert np.max(np.abs(q["ratio"][sel] - orat[sel])) <= 1e-5
    assert np.all(q["ratio"][sel] >= -1e-6) and np.all(q["ratio"][sel] <= 1 + 1e-6)
