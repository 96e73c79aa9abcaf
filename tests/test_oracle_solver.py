"""Solver-level pins for the oracle: closed-form spectra,
brute-force dense eigensolves, eq 3.1 bookkeeping, B-orthonormality, cross-cycle
interlacing, the eq 3.2 subspace rebuilt densely, LOPCG / TRLan reductions and
exact matvec accounting.  None of these reuse oracle code for the expected
value."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest
import scipy.linalg as sla
import scipy.sparse as sp

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _dense_pencil(P):
    A = P.A.to_scipy().toarray()
    B = None if P.B is None else P.B.to_scipy().toarray()
    return A, B


def _resid(A, B, x, th):
    Bx = x if B is None else B @ x
    return np.linalg.norm(A @ x - th * Bx)


# ---------------------------------------------------------------- closed forms
def test_C1_closed_form_tight(orc, gen):
    """C1 at tol_parity 1e-12: eigenvalues 1e-10 relative."""
    P = gen.make("C1")
    r = orc.solve(P.A, None, P.p, P.q, P.l, 1e-12)
    assert r["status"] == "OK"
    ref = np.array(GOLD["C1_eigs"]["values"])
    assert np.max(np.abs(r["eigenvalues"] - ref) / ref) <= 1e-10
    assert np.all(r["residuals"] <= 1e-12)


def test_C1_config_tol_aposteriori(orc, gen):
    """At the config tol the a-posteriori bound |theta - lambda| <= ||r||^2/gap holds."""
    P = gen.make("C1")
    r = orc.solve(P.A, None, P.p, P.q, P.l, P.tol)
    assert r["status"] == "OK" and np.all(r["residuals"] <= P.tol)
    k = np.arange(1, 7)
    lam = 2 - 2 * np.cos(k * np.pi / 1001)
    gaps = np.minimum(np.diff(lam)[:5], np.r_[np.inf, np.diff(lam)[:4]])
    assert np.all(np.abs(r["eigenvalues"] - lam[:5]) <= r["residuals"] ** 2 / gaps * 1.01 + 1e-15)
    # eigenvectors: sin(angle) <= ||r||/gap against the analytic sine vectors
    j = np.arange(1, 1001)
    for i in range(5):
        v = np.sin(j * (i + 1) * np.pi / 1001)
        v /= np.linalg.norm(v)
        s = np.sqrt(max(0.0, 1 - (v @ r["eigenvectors"][:, i]) ** 2))
        assert s <= r["residuals"][i] / gaps[i] * 1.01 + 1e-12


def test_C3_small_clusters_tight(orc, gen):
    """10^3 Laplacian (C3 shape, exact multiplicities 1,3,3,3): p=10 ends on a cluster."""
    P = gen.make("C3", N=10)
    r = orc.solve(P.A, None, 10, 24, 3, 1e-12)
    assert r["status"] == "OK"
    c = 2 - 2 * np.cos(np.arange(1, 11) * np.pi / 11)
    ref = np.sort(np.add.outer(np.add.outer(c, c), c).ravel())[:10]
    assert np.max(np.abs(r["eigenvalues"] - ref) / ref) <= 1e-10
    X = r["eigenvectors"]
    assert np.max(np.abs(X.T @ X - np.eye(10))) <= 1e-12


def test_C4prime_small_pencil_closed_form(orc, gen):
    """d=0 pencil (C4' shape) on 6^3: lambda = (27 - prod(1+2c))/(1 + sum c/6)."""
    P = gen.make("C4", N=6, dscale=0.0)
    r = orc.solve(P.A, P.B, 7, 24, 2, 1e-11)  # ~10 ulp of ||A|| is the residual floor here
    assert r["status"] == "OK"
    c = np.cos(np.arange(1, 7) * np.pi / 7)
    lam = np.sort([(27 - (1 + 2 * a) * (1 + 2 * b) * (1 + 2 * d)) / (1 + (a + b + d) / 6)
                   for a in c for b in c for d in c])[:7]
    assert np.max(np.abs(r["eigenvalues"] - lam) / lam) <= 1e-10


# ---------------------------------------------------------------- brute force
def test_C2_tiny_vs_dense_eigh(orc, gen):
    P = gen.make("C2", N=8)
    A, _ = _dense_pencil(P)
    r = orc.solve(P.A, None, P.p, P.q, P.l, 1e-11)
    assert r["status"] == "OK"
    lam, V = np.linalg.eigh(A)
    assert np.max(np.abs(r["eigenvalues"] - lam[:10]) / lam[:10]) <= 1e-9
    # Weyl: lambda_k(L) <= lambda_k(L+D) <= lambda_k(L) + max d
    L = gen.make("C2", N=8, dscale=0.0)
    lamL = np.linalg.eigh(L.A.to_scipy().toarray())[0][:10]
    assert np.all(lamL <= r["eigenvalues"] + 1e-12) and np.all(r["eigenvalues"] <= lamL + 10.0)
    for i in range(10):
        gap = min(abs(lam[i] - lam[j]) for j in range(len(lam)) if j != i)
        s = np.sqrt(max(0.0, 1 - (V[:, i] @ r["eigenvectors"][:, i]) ** 2))
        assert s <= 1.01 * r["residuals"][i] / gap + 1e-12
        assert _resid(A, None, r["eigenvectors"][:, i], r["eigenvalues"][i]) == pytest.approx(
            r["residuals"][i], rel=1e-6, abs=1e-14)


def test_C4_tiny_pencil_vs_scipy(orc, gen):
    P = gen.make("C4", N=6)
    A, B = _dense_pencil(P)
    r = orc.solve(P.A, P.B, P.p, P.q, P.l, 1e-11)
    assert r["status"] == "OK"
    lam = sla.eigh(A, B, eigvals_only=True)
    assert np.max(np.abs(r["eigenvalues"] - lam[:10]) / lam[:10]) <= 1e-9
    X = r["eigenvectors"]
    assert np.max(np.abs(X.T @ B @ X - np.eye(10))) <= 1e-12
    for i in range(10):  # reported residual is ||A x - theta B x||_2 with ||x||_B = 1 (R15)
        assert _resid(A, B, X[:, i], r["eigenvalues"][i]) == pytest.approx(r["residuals"][i], rel=1e-6, abs=1e-14)
        assert r["residuals"][i] <= 1e-11


# ---------------------------------------------------------------- invariants
def test_bookkeeping_orthonormality_interlacing_accounting(orc, gen):
    P = gen.make("C2", N=6)
    nA = np.linalg.norm(P.A.to_scipy().toarray(), 2)
    ph, m, l = 4, 6, 2
    r = orc.solve(P.A, None, ph, ph + m + l, l, 1e-10, debug=True)
    assert r["status"] == "OK"
    lg = r["log"]
    # eq 3.1 bookkeeping and U^T B U = I at every RR
    assert np.max(lg["terr"]) <= 1e-12 * nA
    assert np.max(lg["orth"]) <= 1e-12
    # cross-cycle interlacing: every kept Ritz value is non-increasing (eq 3.2 contains span X_i)
    th = lg["thetas"]
    assert np.all(th[1:] <= th[:-1] + 1e-14 * np.abs(th[:-1]) + 1e-15 * nA)
    # theta_t monotone while t fixed
    tt, tht = lg["t"], lg["theta_t"]
    same = tt[1:] == tt[:-1]
    assert np.all(tht[1:][same] <= tht[:-1][same] + 1e-14 * nA)
    # exact matvec accounting: init p^ + per cycle m + |X^prev appended| + 1 (+1 per lock with t<=p)
    mv = np.r_[ph, lg["mv"]]
    tnext = np.r_[tt[1:], ph + 1]
    for c in range(len(tt)):
        locks = tnext[c] - tt[c]
        extra = locks if tnext[c] <= ph else locks - 1
        assert mv[c + 1] - mv[c] == m + lg["nprev"][c] + 1 + extra, c
    assert r["a_matvecs"] == mv[-1] + r["verify_matvecs"]
    assert r["verify_matvecs"] == ph  # one verification pass succeeded
    assert r["inner_steps"] == m * len(tt)


def test_frob_tolerance_and_boundary(orc, gen):
    """tol_mode FROB: ||r|| <= tol*||A||_F (eq 5.1); equality passes."""
    P = gen.make("C1", N=200)
    nF = np.sqrt(np.sum(P.A.val ** 2))
    r = orc.solve(P.A, None, 2, 10, 1, 1e-10, tol_mode=1)
    assert r["status"] == "OK" and np.all(r["residuals"] <= 1e-10 * nF)
    g = GOLD["convergence_boundary"]
    assert (g["res"] <= g["normF"] * g["delta"]) == g["converged"]


def test_status_paths(orc, gen):
    P = gen.make("C2", N=6)
    r = orc.solve(P.A, None, 4, 12, 2, 1e-12, max_cycles=2)
    assert r["status"] == "NOT_CONVERGED" and r["cycles"] == 2
    assert np.all(np.isfinite(r["eigenvalues"])) and np.all(r["residuals"] > 0)
    r = orc.solve(P.A, None, 4, 6, 2, 1e-8)  # m = 0
    assert r["status"] == "EINVAL"
    r1 = orc.solve(P.A, None, 4, 12, 2, 1e-10, lock_mode=1)  # WHILE variant, same answer
    r0 = orc.solve(P.A, None, 4, 12, 2, 1e-10)
    assert np.allclose(r1["eigenvalues"], r0["eigenvalues"], rtol=1e-9)


# ------------------------------------------------------ definition of the space
def _rr_dense(A, B, Z, nwant):
    """Dense Rayleigh-Ritz over span(Z): SVD orthonormalisation, then eigh(Q^T A Q, Q^T B Q)."""
    U, s, _ = np.linalg.svd(Z, full_matrices=False)
    Q = U[:, s > 1e-13 * s[0]]
    Bq = Q if B is None else B @ Q
    return sla.eigh(Q.T @ A @ Q, Q.T @ Bq, eigvals_only=True)[:nwant]


def test_subspace_eq32_rebuilt_densely(orc, gen):
    """Per-cycle pin of eq 3.2: span{X_i, u1, C u1, .., C^{m-1} u1, X_{i-1}(:,t..)}
    with C = (I - X X^T B) M (A - rho B), u1 = C x_t -- explicit powers, dense RR."""
    for name in ("C2", "C4"):
        P = gen.make(name, N=4)
        A, B = _dense_pencil(P)
        Bm = np.eye(A.shape[0]) if B is None else B
        Md = 1.0 / np.abs(np.diag(A))
        p, m, l = 3, 3, 2
        r = orc.solve(P.A, P.B, p, p + m + l, l, 1e-13, dump_cycles=6, max_cycles=6)
        d = r["dump"]
        assert np.all(d["t"] == 1)  # no lock in the compared cycles -> X^prev = X_{i-1}(:, 1:l)
        for c in range(len(d["rho"])):
            X, rho = d["X"][c], d["rho"][c]
            C = (np.eye(len(Md)) - X @ X.T @ Bm) @ (Md[:, None] * (A - rho * Bm))
            cols = [X]
            v = C @ X[:, 0]
            for _ in range(m):
                cols.append((v / np.linalg.norm(v))[:, None])
                v = C @ cols[-1][:, 0]
            if c > 0:
                cols.append(d["X"][c - 1][:, :l])
            th = _rr_dense(A, B, np.hstack(cols), p)
            assert np.max(np.abs(th - r["log"]["thetas"][c][:p]) / np.abs(th)) <= 1e-10, (name, c)


def test_lopcg_reduction(orc, gen):
    """m=1, p=l=1, scalar M: span{x_i, r_i, x_{i-1}} = LOPCG (eq 2.2, p=1)."""
    n = 200
    P = gen.make("C1", N=n)
    A = P.A.to_scipy().toarray()
    r = orc.solve(P.A, None, 1, 3, 1, 1e-14, max_cycles=12)
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
        assert abs(w[0] - r["log"]["theta_t"][c]) <= 1e-10 * abs(w[0]), c


def test_trlan_reduction(orc):
    """l=0, M=I, p=1: eq 3.2 degenerates to eq 2.1: RR over
    span{x, r, A r, .., A^{m-1} r}, Laplacian2D(400), first 10 cycles to 1e-8."""
    T = sp.diags([[-1.0] * 19, [2.0] * 20, [-1.0] * 19], [-1, 0, 1])
    A = (sp.kron(T, sp.identity(20)) + sp.kron(sp.identity(20), T)).tocsr()
    Ad = A.toarray()
    m = 4
    r = orc.solve(A, None, 1, 1 + m, 0, 1e-14, max_cycles=10)
    from paper_1711_10128_b200 import inputs
    x = inputs.u01(12, 0, 0, 400)
    x /= np.linalg.norm(x)
    for c in range(10):
        rho = x @ Ad @ x
        v = Ad @ x - rho * x
        cols = [x[:, None]]
        for _ in range(m):
            cols.append((v / np.linalg.norm(v))[:, None])
            v = Ad @ cols[-1][:, 0]
        U, s, _ = np.linalg.svd(np.hstack(cols), full_matrices=False)
        Q = U[:, s > 1e-13 * s[0]]
        w, Y = np.linalg.eigh(Q.T @ Ad @ Q)
        x = Q @ Y[:, 0]
        assert abs(w[0] - r["log"]["theta_t"][c]) <= 1e-8 * abs(w[0]), c


# ------------------------------------------------------------- determinism
def test_determinism_thread_count(tmp_path):
    """Bitwise-identical results for OMP_NUM_THREADS=1 and 8 (blocked fixed-order sums)."""
    code = ("import sys, numpy as np; sys.path.insert(0, %r)\n"
            "import oracle\nfrom paper_1711_10128_b200 import inputs\n"
            "P = inputs.make('C2', N=33)\n"
            "r = oracle.solve(P.A, None, 4, 12, 2, 1e-12, max_cycles=3, want_vectors=False)\n"
            "np.save(sys.argv[1], np.r_[r['eigenvalues'], r['log']['res']])\n") % ROOT
    outs = []
    for th in ("1", "8"):
        f = str(tmp_path / f"o{th}.npy")
        env = dict(os.environ, OMP_NUM_THREADS=th)
        subprocess.check_call([sys.executable, "-c", code, f], env=env)
        outs.append(np.load(f))
    assert np.array_equal(outs[0], outs[1])


def test_closed_form_laplace_basis(gen):
    """tests/closed_form.py (the exact eigenspaces the C3 eigenvector parity is measured against)
    is itself right: A V = V Lambda and V^T V = I on a 12^3 grid, clusters of the sine basis."""
    import sys
    import os
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from closed_form import laplace3d_lowest
    P = gen.make("C3", N=12)
    lam, V, groups = laplace3d_lowest(12, 10)
    A = P.A.to_scipy()
    assert np.max(np.abs(A @ V - V * lam)) <= 1e-14
    assert np.max(np.abs(V.T @ V - np.eye(10))) <= 1e-14
    assert groups == [[0], [1, 2, 3], [4, 5, 6], [7, 8, 9]]
    assert np.allclose(lam, np.linalg.eigvalsh(A.toarray())[:10], rtol=0, atol=1e-13)


def test_trlan_baseline_m_identity(orc, gen):
    """NEXT-4 baseline: precond = none sets M = I (no other change).  With l = 0 and p = 1 the RR
    space of every cycle is thick-restart Lanczos's, eq 2.1: span{x, r, A r, ..,
    A^{m-1} r} -- explicit powers of A, on a NON-constant diagonal (where the Jacobi M would differ
    from I).  With a random block start (p = 3, the paper's rand(n, k)) the Ritz residuals
    are not collinear, so the space is eq 3.2 with M = I: span{X, u1, C u1, ..}, C = (I - X X^T B)
    (A - rho B) -- pinned densely per cycle, also for the pencil C4."""
    P = gen.make("C2", N=5)
    A, _ = _dense_pencil(P)
    m = 4
    r = orc.solve(P.A, None, 1, 1 + m, 0, 1e-13, dump_cycles=6, max_cycles=6, precond=1)
    d = r["dump"]
    for c in range(len(d["rho"])):
        x, rho = d["X"][c][:, 0], d["rho"][c]
        v = A @ x - rho * x
        cols = [x[:, None]]
        for _ in range(m):
            cols.append((v / np.linalg.norm(v))[:, None])
            v = A @ cols[-1][:, 0]
        th = _rr_dense(A, None, np.hstack(cols), 1)
        assert abs(th[0] - r["log"]["thetas"][c][0]) <= 1e-10 * abs(th[0]), c
    for name in ("C2", "C4"):
        P = gen.make(name, N=5)
        A, B = _dense_pencil(P)
        Bm = np.eye(A.shape[0]) if B is None else B
        p = 3
        r = orc.solve(P.A, P.B, p, p + m, 0, 1e-13, dump_cycles=6, max_cycles=6, precond=1)
        d = r["dump"]
        for c in range(len(d["rho"])):
            X, rho, t = d["X"][c], d["rho"][c], d["t"][c]
            C = (np.eye(len(Bm)) - X @ X.T @ Bm) @ (A - rho * Bm)
            cols = [X]
            v = C @ X[:, t - 1]
            for _ in range(m):
                cols.append((v / np.linalg.norm(v))[:, None])
                v = C @ cols[-1][:, 0]
            th = _rr_dense(A, B, np.hstack(cols), p)
            assert np.max(np.abs(th - r["log"]["thetas"][c][:p]) / np.abs(th)) <= 1e-10, (name, c)


@pytest.mark.parametrize("b", [2, 3])
def test_block_trplk_subspace_multishift(orc, gen, b):
    """NEXT-3, block TRPL+K (reading B1): per cycle the RR space is
    span{X, u_0, C u_0, .., u_1, C u_1, ..} -- the block Krylov space of eq 3.2's C =
    (I - X X^T B) M (A - theta_t B) from the seeds u_i = (I - X X^T B) M r_{t+i}, i < b_e =
    min(b, p^ - t + 1) (r_{t+i} with its own Ritz value); the m inner columns are produced
    round-robin (seed i's powers: ceil((m - i) / b_e) columns).  Rebuilt densely from explicit
    powers per cycle (Ritz values = Rayleigh quotients of the dumped X), compared with the oracle's
    Ritz values; also the matvec accounting m + b_e per cycle (+1 per lock) and that b = 1 is
    Algorithm 1 bit for bit."""
    for name in ("C2", "C4"):
        P = gen.make(name, N=5)
        A, B = _dense_pencil(P)
        Bm = np.eye(A.shape[0]) if B is None else B
        Md = 1.0 / np.abs(np.diag(A))
        p, m = 3, 6
        r = orc.solve(P.A, P.B, p, p + m, 0, 1e-13, dump_cycles=5, max_cycles=5, block=b)
        d = r["dump"]
        for c in range(len(d["rho"])):
            X, t = d["X"][c], d["t"][c]
            be = min(b, p - t + 1, m)
            Pj = np.eye(len(Md)) - X @ X.T @ Bm
            cols = [X]
            xt = X[:, t - 1]
            C = Pj @ (Md[:, None] * (A - (xt @ A @ xt) / (xt @ Bm @ xt) * Bm))
            for i in range(be):
                x = X[:, t - 1 + i]
                th = (x @ A @ x) / (x @ Bm @ x)
                Ci = C
                v = Pj @ (Md * (A @ x - th * (Bm @ x)))
                for _ in range(-(-(m - i) // be)):
                    cols.append((v / np.linalg.norm(v))[:, None])
                    v = Ci @ cols[-1][:, 0]
            thr = _rr_dense(A, B, np.hstack(cols), p)
            assert np.max(np.abs(thr - r["log"]["thetas"][c][:p]) / np.abs(thr)) <= 1e-10, (name, b, c)
        lg = r["log"]
        mv = np.diff(np.r_[p, lg["mv"]])
        for c in range(len(mv) - 1):
            # the b_e - 1 extra seed residuals of cycle c were computed at the end of cycle c - 1
            # (cycle 0's from the start-up's A X: no matvec); +1 per lock after the RR
            be = min(b, p - lg["t"][c] + 1, m) if c > 0 else 1
            locks = lg["t"][c + 1] - lg["t"][c]
            assert mv[c] == m + 1 + (be - 1) + locks, (name, b, c)
    P = gen.make("C2", N=8)
    r0 = orc.solve(P.A, None, P.p, P.q, P.l, P.tol, block=0)
    r1 = orc.solve(P.A, None, P.p, P.q, P.l, P.tol, block=1)
    assert np.array_equal(r0["eigenvalues"], r1["eigenvalues"]) and r0["a_matvecs"] == r1["a_matvecs"]


def test_lobpcg_baseline_block_eq22(orc, gen):
    """NEXT-4 baseline: LOBPCG (eq 2.2: "m = p = l") is block TRPL+K with block = p, m = p
    and k_plus = p -- per cycle the RR space span{X_i, M R_i, X_{i-1}} with R_i = A X_i - B X_i Theta_i
    the residuals of all p Ritz vectors and X_{i-1} the previous cycle's Ritz vectors.  Pinned by a
    dense LOBPCG step per cycle (explicit residual block, Jacobi M, SVD orthonormalisation, dense RR)
    while no pair is locked (t = 1), on C2 and the pencil C4."""
    for name in ("C2", "C4"):
        P = gen.make(name, N=5)
        A, B = _dense_pencil(P)
        Bm = np.eye(A.shape[0]) if B is None else B
        Md = 1.0 / np.abs(np.diag(A))
        p = 3
        r = orc.solve(P.A, P.B, p, 3 * p, p, 1e-12, dump_cycles=8, max_cycles=8, block=p)
        d = r["dump"]
        checked = 0
        for c in range(len(d["rho"])):
            if d["t"][c] != 1:
                break
            X = d["X"][c]
            th = np.array([(X[:, j] @ A @ X[:, j]) / (X[:, j] @ Bm @ X[:, j]) for j in range(p)])
            R = A @ X - (Bm @ X) * th
            cols = [X, Md[:, None] * R] + ([d["X"][c - 1]] if c > 0 else [])
            thr = _rr_dense(A, B, np.hstack(cols), p)
            assert np.max(np.abs(thr - r["log"]["thetas"][c][:p]) / np.abs(thr)) <= 1e-10, (name, c)
            checked += 1
        assert checked >= 3


def test_shifted_jacobi_per_cycle(orc, gen):
    """NEXT-2 (per-cycle shift, "M may change at every cycle with the goal to approximate
    (A - rho_i I)^-1", reading P2c): precond = 2 re-forms the Jacobi M of A - rho_i B with the
    cycle's shift; pinned by the eq 3.2 space rebuilt densely with that M, per cycle, C2 and C4."""
    for name in ("C2", "C4"):
        P = gen.make(name, N=4)
        A, B = _dense_pencil(P)
        Bm = np.eye(A.shape[0]) if B is None else B
        p, m, l = 3, 3, 2
        r = orc.solve(P.A, P.B, p, p + m + l, l, 1e-13, dump_cycles=6, max_cycles=6, precond=2)
        d = r["dump"]
        assert np.all(d["t"] == 1)
        for c in range(len(d["rho"])):
            X, rho = d["X"][c], d["rho"][c]
            Md = 1.0 / np.maximum(np.abs(np.diag(A) - rho * np.diag(Bm)), 1e-8 * np.max(np.abs(np.diag(A))))
            C = (np.eye(len(Md)) - X @ X.T @ Bm) @ (Md[:, None] * (A - rho * Bm))
            cols = [X]
            v = C @ X[:, 0]
            for _ in range(m):
                cols.append((v / np.linalg.norm(v))[:, None])
                v = C @ cols[-1][:, 0]
            if c > 0:
                cols.append(d["X"][c - 1][:, :l])
            th = _rr_dense(A, B, np.hstack(cols), p)
            assert np.max(np.abs(th - r["log"]["thetas"][c][:p]) / np.abs(th)) <= 1e-10, (name, c)


def test_ic0_preconditioned_space(orc, gen):
    """NEXT-2, IC(0) (precond = 3, reading P2a): eq 3.2's space per cycle with M = (L L^T)^-1,
    L = the oracle's IC(0) factor (pinned in test_oracle_branches.py), rebuilt densely, C2 and C4."""
    for name in ("C2", "C4"):
        P = gen.make(name, N=4)
        A, B = _dense_pencil(P)
        Bm = np.eye(A.shape[0]) if B is None else B
        L = orc.ic0(P.A, P.B, 0.0).toarray()
        Mfull = np.linalg.inv(L @ L.T)
        p, m, l = 3, 3, 2
        r = orc.solve(P.A, P.B, p, p + m + l, l, 1e-13, dump_cycles=6, max_cycles=6, precond=3)
        d = r["dump"]
        # the first 4 cycles: IC(0) converges fast, and once the residual is tiny the explicit
        # power basis of the dense rebuild loses its conditioning (not the oracle's orthogonalised one)
        for c in range(min(4, len(d["rho"]))):
            if d["t"][c] != 1:
                break
            X, rho = d["X"][c], d["rho"][c]
            C = (np.eye(len(A)) - X @ X.T @ Bm) @ (Mfull @ (A - rho * Bm))
            cols = [X]
            v = C @ X[:, 0]
            for _ in range(m):
                cols.append((v / np.linalg.norm(v))[:, None])
                v = C @ cols[-1][:, 0]
            if c > 0:
                cols.append(d["X"][c - 1][:, :l])
            th = _rr_dense(A, B, np.hstack(cols), p)
            assert np.max(np.abs(th - r["log"]["thetas"][c][:p]) / np.abs(th)) <= 1e-10, (name, c)
