"""The GPU solve in the paper's limiting cases (SURVEY 8(c.4) reductions), checked against the
dense construction of the method each case reduces to -- not against the oracle:
  * m = 1, p = l = 1, scalar M: the cycle is LOPCG, RR over span{x_i, r_i, x_{i-1}} (eq 2.2,
    P:80);
  * l = 0, M = I (constant diagonal), p = 1: eq 3.2 degenerates to thick-restart Lanczos,
    RR over span{x, r, A r, .., A^{m-1} r} (eq 2.1)."""
import numpy as np
import pytest
import scipy.sparse as sp

from gpu_util import need_gpu

pytestmark = pytest.mark.gpu


def _gpu_log(trplk, A, p, q, l, tol, cycles):
    ctx = trplk.trplk_create(A, None, 0.0)
    trplk.trplk_solve(ctx, p, q, l, tol, max_cycles=cycles)
    log = trplk.trplk_get_log(ctx, ph=p)
    ctx.close()
    return log


def test_lopcg_reduction_gpu(gen):
    torch, trplk = need_gpu()
    n = 200
    P = gen.make("C1", N=n)
    A = P.A.to_scipy().toarray()
    log = _gpu_log(trplk, P.A, 1, 3, 1, 1e-14, 12)
    x = gen.u01(12, 0, 0, n)
    x /= np.linalg.norm(x)
    xprev = None
    for c in range(12):
        rho = x @ A @ x
        res = A @ x - rho * x
        cols = [x[:, None], res[:, None]] + ([xprev[:, None]] if xprev is not None else [])
        U, s, _ = np.linalg.svd(np.hstack(cols), full_matrices=False)
        Q = U[:, s > 1e-13 * s[0]]
        w, Y = np.linalg.eigh(Q.T @ A @ Q)
        xprev, x = x, Q @ Y[:, 0]
        assert abs(w[0] - log["theta_t"][c]) <= 1e-10 * abs(w[0]), c


@pytest.mark.parametrize("N", [20, 64])
def test_trlan_reduction_gpu(gen, N):
    """N = 20 (400 rows) and N = 64 (4,096 rows): both run the single-CTA inner loop
    (q = 5 <= 24); the multi-kernel path is covered by the oracle parity tests."""
    torch, trplk = need_gpu()
    T = sp.diags([[-1.0] * (N - 1), [2.0] * N, [-1.0] * (N - 1)], [-1, 0, 1])
    A = (sp.kron(T, sp.identity(N)) + sp.kron(sp.identity(N), T)).tocsr()
    m = 4
    log = _gpu_log(trplk, A, 1, 1 + m, 0, 1e-14, 10)
    n = N * N
    x = gen.u01(12, 0, 0, n)
    x /= np.linalg.norm(x)
    for c in range(10):
        Ax = A @ x
        rho = x @ Ax
        v = Ax - rho * x
        cols = [x[:, None]]
        for _ in range(m):
            cols.append((v / np.linalg.norm(v))[:, None])
            v = A @ cols[-1][:, 0]
        U, s, _ = np.linalg.svd(np.hstack(cols), full_matrices=False)
        Q = U[:, s > 1e-13 * s[0]]
        AQ = A @ Q
        w, Y = np.linalg.eigh(Q.T @ AQ)
        x = Q @ Y[:, 0]
        assert abs(w[0] - log["theta_t"][c]) <= 1e-8 * abs(w[0]), c
