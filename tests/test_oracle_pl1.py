"""Pins of the PL+1 oracle (Algorithm 2; NEXT-1 of SURVEY 8(f)).

Every expected value comes from something other than the oracle: closed-form spectra, dense
(scipy) generalized eigensolves, Rayleigh-Ritz over explicitly built subspaces (Krylov powers,
the quasi-optimal space U_2 of section 4.3), and the algebraic identities the paper states
(monotone rho, exact step-7 conjugacy)."""
import numpy as np
import pytest
import scipy.linalg as sla
import scipy.sparse as sp


def _csr_dense(D):
    return sp.csr_matrix(D)


def _min_rq(A, B, V):
    """Lowest Ritz value of the pencil (A, B) on range(V) (dense, orthonormalised basis)."""
    Q, _ = np.linalg.qr(V)
    H = Q.T @ A @ Q
    S = Q.T @ (Q if B is None else B @ Q)
    return sla.eigh(0.5 * (H + H.T), 0.5 * (S + S.T), eigvals_only=True)[0]


def _jacobi(A, B, sigma):
    """M of reading R1 written out in numpy: 1 / max(|a_ii - sigma b_ii|, 1e-8 max_j |a_jj|)."""
    a = np.diag(A)
    b = np.ones_like(a) if B is None else np.diag(B)
    return 1.0 / np.maximum(np.abs(a - sigma * b), 1e-8 * np.max(np.abs(a)))


def _rq(A, B, x):
    return float(x @ A @ x) / float(x @ (x if B is None else B @ x))


def test_exact_start_converges_at_k0(orc):
    """SPEC example: A = diag(1,2,3), B = I, M = I, x_0 = v_1 -> converged at k = 0, rho = 1."""
    A = _csr_dense(np.diag([1.0, 2.0, 3.0]))
    r = orc.pl1_solve(A, None, m=1, tol=1e-12, x0=np.array([1.0, 0.0, 0.0]), use_precond=False)
    assert r["status"] == "OK" and r["cycles"] == 0
    assert r["rho"] == 1.0
    assert r["a_matvecs"] == 1


def test_laplacian_closed_form(orc, gen):
    """3D Laplacian 10^3 (C3 shape, d = 0): lambda_1 = 3 (2 - 2 cos(pi/11))."""
    P = gen.make("C3", N=10)
    r = orc.pl1_solve(P.A, None, m=4, tol=1e-10, sigma=P.sigma)
    lam = 3 * (2 - 2 * np.cos(np.pi / 11))
    assert r["status"] == "OK"
    assert abs(r["rho"] - lam) <= 1e-12 * lam
    assert r["residual"] <= 1e-10


@pytest.mark.parametrize("variant", [0, 1])
def test_dense_pencil(orc, variant):
    """Random symmetric A, SPD B (n = 80): rho -> lambda_1 of scipy's eigh(A, B); x is
    B-normalised and B-aligned with v_1.  Both step-7 variants (paper, practical P:281)."""
    rng = np.random.default_rng(5)
    n = 80
    X = rng.standard_normal((n, n))
    A = 0.5 * (X + X.T) + np.diag(np.linspace(1, 30, n))
    Y = rng.standard_normal((n, n)) / np.sqrt(n)
    B = Y @ Y.T + np.eye(n)
    lam, V = sla.eigh(A, B)
    r = orc.pl1_solve(_csr_dense(A), _csr_dense(B), m=3, tol=1e-10, sigma=lam[0] - 1.0, variant=variant)
    assert r["status"] == "OK"
    assert abs(r["rho"] - lam[0]) <= 1e-10 * abs(lam[0])
    x = r["x"]
    assert abs(x @ B @ x - 1) <= 1e-12
    assert abs(abs(x @ B @ V[:, 0]) - 1) <= 1e-9
    assert np.linalg.norm(A @ x - r["rho"] * (B @ x)) <= 1e-10 * (1 + 1e-6)


@pytest.mark.parametrize("name,N", [("C2", 10), ("C4", 6)])
def test_monotone_rho_and_step7_conjugacy(orc, gen, name, N):
    """rho_{k+1} <= rho_k (the RR space contains x_k) and the step-7 identity
    p_{k-1}^T (A - rho_{k-1} B) p_k = 0 (Lemma 8's proof) to 1e-10 ||A||_F on every iteration."""
    P = gen.make(name, N=N)
    r = orc.pl1_solve(P.A, P.B, m=4, tol=1e-9, sigma=P.sigma)
    assert r["status"] == "OK"
    rho = r["log"]["rho"]
    assert np.all(np.diff(rho) <= 1e-13 * np.abs(rho[1:]))
    assert np.max(np.abs(r["log"]["conj"])) <= 1e-10
    # the Ritz value of step 5 is the Rayleigh quotient of the next iterate (step 6)
    ritz = r["log"]["ritz"][:-1]
    assert np.max(np.abs(ritz - rho[1:]) / np.abs(rho[1:])) <= 1e-12
    # dense lambda_1
    A = P.A.to_scipy().toarray()
    B = None if P.B is None else P.B.to_scipy().toarray()
    lam = sla.eigh(A, B, eigvals_only=True)[0]
    assert abs(r["rho"] - lam) <= 1e-11 * abs(lam)


def test_first_iteration_is_rr_on_krylov_powers(orc, gen):
    """Step 4 (P1) + step 5 at k = 0: x_1 is the Ritz vector of span{x_0, M(A-rho_0 B)x_0, ...,
    [M(A-rho_0 B)]^m x_0} -- the space rebuilt here from explicit powers (no oracle code)."""
    P = gen.make("C4", N=6)
    A = P.A.to_scipy().toarray()
    B = P.B.to_scipy().toarray()
    m = 3
    Mv = _jacobi(A, B, P.sigma)
    n = A.shape[0]
    x0 = np.random.default_rng(3).random(n)
    x0 /= np.sqrt(x0 @ B @ x0)
    rho0 = _rq(A, B, x0)
    K = [x0]
    for _ in range(m):
        K.append(Mv * ((A - rho0 * B) @ K[-1]))
    ref = _min_rq(A, B, np.column_stack(K))
    r = orc.pl1_solve(P.A, P.B, m=m, tol=1e-300, sigma=P.sigma, max_cycles=1, x0=x0)
    assert r["status"] == "NOT_CONVERGED" and r["cycles"] == 1
    assert abs(r["log"]["rho"][0] - rho0) <= 1e-13 * rho0
    assert abs(r["rho"] - ref) <= 1e-12 * abs(ref)
    assert abs(_rq(A, B, r["x"]) - ref) <= 1e-12 * abs(ref)
    assert r["a_matvecs"] == 1 + m + 1  # x_0, A g_1..g_m, A x_1 (P5)


def test_x2_is_global_minimizer_in_U2(orc, gen):
    """Section 4.3 (m = 1): x_2 is extracted from span{x_1, g_1, p_0} = U_2 = span{x_0} + W_2,
    W_2 = span{g_0, g_1} = span{M r_0, M r_1} -- so rho(x_2) is the minimum of the Rayleigh
    quotient over U_2 (quasi-optimality ratio 0 at k <= 2, SPEC pl1_analysis)."""
    P = gen.make("C2", N=10)
    A = P.A.to_scipy().toarray()
    Mv = _jacobi(A, None, P.sigma)
    n = A.shape[0]
    x0 = np.random.default_rng(4).random(n)
    x0 /= np.linalg.norm(x0)
    r1 = orc.pl1_solve(P.A, None, m=1, tol=1e-300, sigma=P.sigma, max_cycles=1, x0=x0)
    r2 = orc.pl1_solve(P.A, None, m=1, tol=1e-300, sigma=P.sigma, max_cycles=2, x0=x0)
    x1 = r1["x"]
    res0 = A @ x0 - _rq(A, None, x0) * x0
    res1 = A @ x1 - _rq(A, None, x1) * x1
    ref = _min_rq(A, None, np.column_stack([x0, Mv * res0, Mv * res1]))
    assert abs(r2["rho"] - ref) <= 1e-12 * abs(ref)
    # and x_3 is not worse than the minimiser over U_3 by more than rounding (ratio >= 0)
    r3 = orc.pl1_solve(P.A, None, m=1, tol=1e-300, sigma=P.sigma, max_cycles=3, x0=x0)
    x2 = r2["x"]
    res2 = A @ x2 - _rq(A, None, x2) * x2
    ref3 = _min_rq(A, None, np.column_stack([x0, Mv * res0, Mv * res1, Mv * res2]))
    assert r3["rho"] >= ref3 - 1e-12 * abs(ref3)


def test_matvec_accounting(orc, gen):
    """P5: A-matvecs = 1 + per iteration m + 1 + [k > 0] (no breakdowns on C2)."""
    P = gen.make("C2", N=10)
    m = 4
    r = orc.pl1_solve(P.A, None, m=m, tol=1e-9, sigma=P.sigma)
    K = r["cycles"]
    assert np.all(r["log"]["mg"][:K] == m)
    assert r["a_matvecs"] == 1 + K * (m + 1) + (K - 1)


# ---------------------------------------------------------------- quasi-optimality diagnostic (P7)
# Definition defnglbopt: rho(y*_k) = min of the Rayleigh quotient over
# U_k = span{x_0} + span{g_0, ..., g_{k-1}}.


def test_qopt_brute_force_generalized(orc, gen):
    """rho(y*_k) of the oracle = the lowest Ritz value of (A, B) on the explicitly stacked
    [x_0, g_0, ..., g_{k-1}] (numpy QR + scipy generalized eigh), C4-shaped pencil (B != I)."""
    P = gen.make("C4", N=6)
    A = P.A.to_scipy().toarray()
    B = P.B.to_scipy().toarray()
    n = A.shape[0]
    x0 = np.random.default_rng(7).random(n)
    cap = 10
    r = orc.pl1_solve(P.A, P.B, m=2, tol=1e-300, sigma=P.sigma, max_cycles=cap - 1, x0=x0,
                      qopt_cap=cap, want_g=True)
    q, dim, G = r["log"]["qopt"], r["log"]["qdim"], r["g"]
    assert len(q) == cap and G.shape == (n, cap - 1)
    assert np.array_equal(dim, np.arange(1, cap + 1))
    for k in range(cap):
        ref = _min_rq(A, B, np.column_stack([x0] + [G[:, j] for j in range(k)]))
        assert abs(q[k] - ref) <= 1e-10 * abs(ref), (k, q[k], ref)


@pytest.mark.parametrize("m", [1, 3])
def test_qopt_special_cases(orc, gen, m):
    """rho(y*_0) = rho_0 (U_0 = span{x_0}); x_1 is the RR minimiser over span{x_0, G_0} which
    contains U_1, so rho(y*_1) = rho_1; for m = 1, U_2 = span{x_1, g_1, p_0} (section 4.3), so
    rho(y*_2) = rho_2; always lambda_1 <= rho(y*_k) <= rho_k and rho(y*_k) nonincreasing.  The
    diagnostic leaves the trajectory and the matvec counts untouched."""
    P = gen.make("C2", N=8)
    A = P.A.to_scipy().toarray()
    lam1 = np.linalg.eigvalsh(A)[0]
    base = orc.pl1_solve(P.A, None, m=m, tol=1e-9, sigma=P.sigma)
    r = orc.pl1_solve(P.A, None, m=m, tol=1e-9, sigma=P.sigma, qopt_cap=64)
    assert r["a_matvecs"] == base["a_matvecs"] and r["b_matvecs"] == base["b_matvecs"]
    assert np.array_equal(r["log"]["rho"], base["log"]["rho"])
    rho, q = r["log"]["rho"], r["log"]["qopt"]
    K = len(q)
    assert K == min(len(rho), 64) and K >= 4
    eps = 1e-13 * abs(lam1)
    assert abs(q[0] - rho[0]) <= eps
    assert abs(q[1] - rho[1]) <= eps
    if m == 1:
        assert abs(q[2] - rho[2]) <= eps
    assert np.all(q <= rho[:K] + eps) and np.all(q >= lam1 - eps)
    assert np.all(np.diff(q) <= eps)


def test_qopt_full_space(orc):
    """Dense n = 6, m = 1: once dim U_k = n, rho(y*_k) = lambda_1 to rounding, and later g_k
    (inside U_k) are dropped by the R16 dependence test so dim U_k stays n."""
    rng = np.random.default_rng(11)
    n = 6
    Q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    lam = np.array([1.0, 1.5, 2.0, 3.0, 5.0, 8.0])
    A = Q @ np.diag(lam) @ Q.T
    A = 0.5 * (A + A.T)
    r = orc.pl1_solve(_csr_dense(A), None, m=1, tol=1e-300, max_cycles=12, use_precond=False,
                      x0=rng.random(n), qopt_cap=13)
    q, dim = r["log"]["qopt"], r["log"]["qdim"]
    full = np.nonzero(dim == n)[0]
    assert len(full) >= 2 and np.all(dim <= n) and np.all(np.diff(dim) >= 0)
    assert np.all(np.abs(q[full] - lam[0]) <= 1e-13 * lam[0])
