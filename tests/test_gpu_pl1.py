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
