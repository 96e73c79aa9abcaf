"""Pins of the oracle's rarely taken branches (VERDICT r01 "parity unpinned" items), each against
a closed form or a dimension count -- not against the oracle itself.

R3: CGS2 takes a third pass iff pass 2 kept less than 1/sqrt2 of the
norm; R3/R16: breakdown iff the final B-norm < 1e-14 x the input norm; R16 (S:257-258,
S:266): an inner Krylov breakdown ends the inner loop with the columns built so far, a seed in
span(X) is replaced by a stream-2 random vector, a dependent X^prev column is dropped.
"""
import numpy as np
import pytest
import scipy.sparse as sp


def _frame(n, k, eta, seed=3):
    """Orthonormal q_0..q_k (numpy QR) and V = [v_1, v_2, q_2..q_{k-1}] with v_1 = q_0,
    v_2 = eta q_0 + sqrt(1 - eta^2) q_1 (unit columns, v_1^T v_2 = eta, all others orthonormal);
    e = q_k is orthogonal to every column of V."""
    Q, _ = np.linalg.qr(np.random.default_rng(seed).standard_normal((n, k + 1)))
    V = Q[:, :k].copy(order="F")
    V[:, 1] = eta * Q[:, 0] + np.sqrt(1.0 - eta * eta) * Q[:, 1]
    return V, Q[:, k]


@pytest.mark.parametrize("eta,gamma", [(0.5, 0.1), (1e-4, 1e-5), (0.3, 0.05)])
def test_cgs2_third_pass_closed_form(orc, eta, gamma):
    """w = v_1 + gamma e against V (v_1^T v_2 = eta).  Exact passes:
       pass 1: coefficients (1, eta)      -> w' = gamma e - eta v_2,          ||w'||^2 = gamma^2 + eta^2
       pass 2: coefficients (-eta^2, -eta) -> w'' = gamma e + eta^2 v_1,     ||w''||^2 = gamma^2 + eta^4
       gamma^2 < eta^2 - 2 eta^4  <=>  ||w''|| < ||w'|| / sqrt2  -> third pass:
       pass 3: coefficients (eta^2, eta^3) -> w''' = gamma e - eta^3 v_2,   ||w'''||^2 = gamma^2 + eta^6
    Summed coefficients h = (1, eta^3, 0, ...)."""
    n, k = 300, 6
    assert gamma ** 2 < eta ** 2 - 2 * eta ** 4
    V, e = _frame(n, k, eta)
    w0 = V[:, 0] + gamma * e
    w, h, beta, brk, passes = orc.cgs2(V, w0)
    assert passes == 3 and not brk
    assert abs(beta - np.sqrt(gamma ** 2 + eta ** 6)) <= 1e-13
    assert np.max(np.abs(w - (gamma * e - eta ** 3 * V[:, 1]))) <= 1e-14
    href = np.zeros(k)
    href[0], href[1] = 1.0, eta ** 3
    assert np.max(np.abs(h - href)) <= 1e-14


def test_cgs2_third_pass_threshold_boundary(orc):
    """Either side of gamma^2 = eta^2 - 2 eta^4 (eta = 0.5: 0.125): 2 passes above, 3 below."""
    n, k, eta = 300, 4, 0.5
    V, e = _frame(n, k, eta, seed=5)
    for gamma, want in ((np.sqrt(0.125) * 1.01, 2), (np.sqrt(0.125) * 0.99, 3)):
        w, h, beta, brk, passes = orc.cgs2(V, V[:, 0] + gamma * e)
        assert passes == want and not brk
        ref = np.sqrt(gamma ** 2 + (eta ** 4 if want == 2 else eta ** 6))
        assert abs(beta - ref) <= 1e-13


@pytest.mark.parametrize("delta,brk_want", [(1e-17, True), (1e-12, False)])
def test_cgs2_breakdown_threshold(orc, delta, brk_want):
    """w = V c + delta e with orthonormal V: the B-norm after CGS2 is delta (up to rounding
    ~1e-16 ||V c||); breakdown iff delta < 1e-14 ||w|| (R3/R16)."""
    n, k = 500, 8
    Q, _ = np.linalg.qr(np.random.default_rng(7).standard_normal((n, k + 1)))
    V, e = np.asfortranarray(Q[:, :k]), Q[:, k]
    c = np.random.default_rng(8).standard_normal(k)
    w0 = V @ c + delta * np.linalg.norm(c) * e
    w, h, beta, brk, passes = orc.cgs2(V, w0)
    assert brk == brk_want
    if not brk_want:
        assert abs(beta - delta * np.linalg.norm(c)) <= 1e-3 * delta * np.linalg.norm(c)
        assert np.max(np.abs(h - c)) <= 1e-13 * np.linalg.norm(c)


def _diag3(reps=20):
    """A = diag(1, 2, 3) with each value repeated: every Krylov space K(A, x) has dimension <= 3."""
    return sp.diags(np.repeat([1.0, 2.0, 3.0], reps)).tocsr()


def test_inner_krylov_breakdown_dimension_count(orc):
    """p = 1: span{x, u_1, C u_1, ...} with C = (I - x x^T) M (A - rho I) (eq 3.2) lies in the
    A-invariant space span{x, A x, A^2 x}, of dimension 3 (three distinct eigenvalues, x random):
    the inner loop breaks down after 2 Krylov columns (R16), the basis has exactly 3 columns, the
    Rayleigh-Ritz on an invariant subspace is exact: theta_1 = lambda_1 = 1, residual at rounding
    level, one cycle, A-matvecs = 1 (start) + 2 (inner) + 1 (residual) + 1 (verification)."""
    r = orc.solve(_diag3(), None, p=1, q=8, l=0, tol=1e-8)
    assert r["status"] == "OK" and r["cycles"] == 1
    assert list(r["log"]["k"]) == [3]
    assert abs(r["eigenvalues"][0] - 1.0) <= 1e-14
    assert r["residuals"][0] <= 1e-13
    assert r["a_matvecs"] == 5 and r["inner_steps"] == 2


def test_inner_breakdown_full_space_exact_rr(orc):
    """n = p^ + 1: the seed completes R^n, so the first inner CGS2 (j = 1 < m = 2) breaks down
    whatever the vector, and the RR on R^n returns the exact spectrum (LAPACK) in one cycle."""
    rng = np.random.default_rng(11)
    R = rng.standard_normal((6, 6))
    A = sp.csr_matrix(R + R.T + 8 * np.eye(6))
    r = orc.solve(A, None, p=5, q=7, l=0, tol=1e-8, lock_mode=1)
    assert r["status"] == "OK" and r["cycles"] == 1 and list(r["log"]["k"]) == [6]
    assert np.max(np.abs(r["eigenvalues"] - np.linalg.eigvalsh(A.toarray())[:5])) <= 1e-13


def test_seed_in_span_X_random_replacement(orc):
    """A = I: every start vector is an eigenvector, the residual of the target lies in span(X)
    (it is zero up to rounding along x_t), so the seed CGS2 breaks down and a stream-2 random
    vector replaces it (R16); the solve still ends with theta = 1 and B-orthonormal X."""
    r = orc.solve(sp.identity(40, format="csr"), None, p=2, q=6, l=1, tol=1e-8)
    assert r["status"] == "OK"
    assert r["random_draws"] >= 1
    assert np.max(np.abs(r["eigenvalues"] - 1.0)) <= 1e-14
    X = r["eigenvectors"]
    assert np.max(np.abs(X.T @ X - np.eye(2))) <= 1e-13


def test_dependent_xprev_dropped(orc):
    """diag(1,2,3) x 20, p = 2, l = 1, unreachable tol: once the two Ritz vectors span the
    2-dimensional lambda = 1 part of the invariant space S = span{x_i, A x_i, A^2 x_i}, the X^prev
    column (a vector of that part) lies in span(X) and is dropped (R16) in every later cycle --
    the log shows 0 appended columns where the target t is unchanged and l = 1 would append one;
    the matvec count is m + appended + 1 per cycle."""
    r = orc.solve(_diag3(), None, p=2, q=9, l=1, tol=1e-30, max_cycles=4)
    lg = r["log"]
    assert r["status"] == "NOT_CONVERGED"
    assert list(lg["t"]) == [1, 1, 1, 1]
    assert list(lg["nprev"][2:]) == [0, 0]  # X^prev offered (t unchanged, l = 1), dropped
    assert np.max(np.abs(r["eigenvalues"] - 1.0)) <= 1e-14
    mv = np.diff(np.r_[2, lg["mv"]])  # start-up: p^ = 2 matvecs
    G = lg["k"] - 2 - lg["nprev"]
    assert np.array_equal(mv, G + lg["nprev"] + 1)


def test_inner_steps_entry_matches_bookkeeping(orc, gen):
    """orc_inner_steps (bench.py's oracle sample): from an orthonormal U(:, :k0) the new columns
    are orthonormal against it and T = U^T A U on the columns it filled (eq 3.1)."""
    P = gen.make("C2", N=10)
    n = P.A.n
    k0, s = 6, 4
    Q, _ = np.linalg.qr(np.random.default_rng(2).standard_normal((n, k0)))
    U = np.zeros((n, k0 + s), order="F")
    U[:, :k0] = Q
    M = orc.jacobi_diag(P.A)
    done, T = orc.inner_steps(P.A, None, M, 2.5, U, k0, s)
    assert done == s
    assert np.max(np.abs(U.T @ U - np.eye(k0 + s))) <= 1e-13
    AU = P.A.to_scipy() @ U
    for j in range(k0 - 1, k0 + s - 1):  # columns k0-1 .. k0+s-2 had their T column filled
        assert np.max(np.abs(T[: j + 1, j] - U[:, : j + 1].T @ AU[:, j])) <= 1e-12


@pytest.mark.parametrize("cfg,N", [("C2", 6), ("C4", 5), ("C3", 7)])
def test_ic0_defining_property(orc, gen, cfg, N):
    """NEXT-2, IC(0) of K = A - sigma B (reading P2a): L has K's lower pattern and (L L^T)_ij =
    K_ij on that pattern -- the definition of the no-fill incomplete Cholesky factor; outside the
    pattern L L^T carries the dropped fill."""
    P = gen.make(cfg, N=N)
    sigma = 0.7
    L = orc.ic0(P.A, P.B, sigma)
    A = P.A.to_scipy().toarray()
    K = A - sigma * (np.eye(len(A)) if P.B is None else P.B.to_scipy().toarray())
    Ld = L.toarray()
    assert np.array_equal(Ld != 0, np.tril(A) != 0)
    LL = Ld @ Ld.T
    on = np.tril(A) != 0
    assert np.max(np.abs(LL - K)[on]) <= 1e-13 * np.max(np.abs(K))


def test_ic0_tridiagonal_is_cholesky_and_solve(orc, gen):
    """For a tridiagonal matrix IC(0) drops nothing: L L^T = A (numpy Cholesky), and the IC(0)
    preconditioned solve is exact -- the C1 oracle converges in a handful of cycles."""
    P = gen.make("C1", N=60)
    L = orc.ic0(P.A).toarray()
    A = P.A.to_scipy().toarray()
    assert np.max(np.abs(L - np.linalg.cholesky(A))) <= 1e-14
    r = orc.solve(P.A, None, 3, 10, 1, 1e-10, precond=3)
    assert r["status"] == "OK"
    c = 2 - 2 * np.cos(np.arange(1, 4) * np.pi / 61)
    assert np.max(np.abs(r["eigenvalues"] - c) / c) <= 1e-9
