"""Pins for the oracle's primitives against things other than the oracle itself
(SURVEY 8(c.4)): printed worked examples (tests/golden/spec_examples.json),
analytic eigenvectors, math.fsum, LAPACK via numpy, constructed projections."""
import json
import math
import os

import numpy as np
import pytest
import scipy.sparse as sp

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def _csr_of_dense(D):
    return sp.csr_matrix(np.asarray(D, dtype=np.float64))


# ------------------------------------------------------------------ RNG (R13)
def test_rng_matches_inputs_module_and_is_uniform(orc, gen):
    # two independent implementations of the stated counter-based generator agree
    xs = gen.u01(12, 0, 0, 4096)
    ys = np.array([orc.u01(12, 0, i) for i in range(4096)])
    assert np.array_equal(xs, ys)
    big = gen.u01(12, 1, 0, 200_000)
    assert big.min() >= 0.0 and big.max() < 1.0
    assert abs(big.mean() - 0.5) < 5e-3
    assert abs(big.var() - 1.0 / 12) < 2e-3
    # streams and seeds decorrelate
    assert abs(np.corrcoef(gen.u01(12, 0, 0, 50000), gen.u01(12, 1, 0, 50000))[0, 1]) < 0.02
    assert not np.array_equal(gen.u01(12, 0, 0, 16), gen.u01(13, 0, 0, 16))


# ---------------------------------------------------------------- SpMV (S1)
def test_spmv_spec_examples(orc):
    g = GOLD["spmv_tridiag3"]
    A = sp.diags([[-1.0] * 2, [2.0] * 3, [-1.0] * 2], [-1, 0, 1]).tocsr()
    assert np.array_equal(orc.spmv(A, g["x"]), np.array(g["y"], float))
    g = GOLD["spmv_identity"]
    assert np.array_equal(orc.spmv(sp.identity(3, format="csr"), g["x"]), np.array(g["y"], float))


def test_spmv_vs_dense_random(orc):
    rng = np.random.default_rng(0)
    for n in (1, 7, 64, 200):
        R = sp.random(n, n, density=0.1, random_state=rng.integers(1 << 30)) + sp.identity(n)
        A = (R + R.T).tocsr()
        x = rng.standard_normal(n)
        y = orc.spmv(A, x)
        yd = A.toarray() @ x
        assert np.max(np.abs(y - yd)) <= 1e-13 * max(1.0, np.max(np.abs(yd)))


def test_spmv_analytic_eigenvectors(orc, gen):
    # 1-D: sin(j k pi/(n+1)) with lambda = 2-2cos(k pi/(n+1))
    n = 1000
    A = gen.make("C1").A
    j = np.arange(1, n + 1)
    for k in (1, 2, 500):
        v = np.sin(j * k * np.pi / (n + 1))
        lam = 2 - 2 * np.cos(k * np.pi / (n + 1))
        assert np.max(np.abs(orc.spmv(A, v) - lam * v)) <= 1e-13 * np.max(np.abs(v)) * 4
    # 3-D 7-pt Laplacian, 27-pt A0 = 27I - T1xT1xT1, mass B = I + adj7/12: sine tensor basis
    N = 10
    s = [np.sin(np.arange(1, N + 1) * kk * np.pi / (N + 1)) for kk in range(1, N + 1)]
    c = [np.cos(kk * np.pi / (N + 1)) for kk in range(1, N + 1)]
    for (a, b, d) in [(0, 0, 0), (1, 0, 2), (4, 7, 9)]:
        v = np.einsum("i,j,k->kji", s[a], s[b], s[d]).ravel()  # x fastest
        L7 = gen.stencil(3, 7, N, 6.0, -1.0).to_scipy()
        lam = sum(2 - 2 * cc for cc in (c[a], c[b], c[d]))
        assert np.max(np.abs(orc.spmv(L7, v) - lam * v)) <= 1e-13 * 12
        A27 = gen.stencil(3, 27, N, 26.0, -1.0).to_scipy()
        lam = 27 - (1 + 2 * c[a]) * (1 + 2 * c[b]) * (1 + 2 * c[d])
        assert np.max(np.abs(orc.spmv(A27, v) - lam * v)) <= 1e-13 * 54
        B7 = gen.stencil(3, 7, N, 1.0, 1.0 / 12).to_scipy()
        lam = 1 + (c[a] + c[b] + c[d]) / 6
        assert np.max(np.abs(orc.spmv(B7, v) - lam * v)) <= 1e-13 * 2


def test_generated_matrices_symmetric_sorted(gen):
    for name, N in (("C2", 6), ("C4", 5), ("C1", None)):
        P = gen.make(name, N=N)
        for M in (P.A, P.B):
            if M is None:
                continue
            S = M.to_scipy()
            assert abs(S - S.T).max() == 0.0
            for i in range(M.rows):
                cols = M.col[M.rowptr[i]:M.rowptr[i + 1]]
                assert np.all(np.diff(cols) > 0)
                assert i in cols  # diagonal stored


def test_nnz_formulas(gen):
    # nnz(7-pt) = N^3 + 6(N-1)N^2; nnz(27-pt) = (3N-2)^3
    for N in (4, 9):
        assert gen.stencil(3, 7, N, 6, -1).nnz == N ** 3 + 6 * (N - 1) * N ** 2
        assert gen.stencil(3, 27, N, 26, -1).nnz == (3 * N - 2) ** 3


def test_slab_generation_matches_global(gen):
    P = gen.make("C2", N=6)
    n = P.A.n
    for nr in (2, 3):
        for r in range(nr):
            b, e = gen.slab_rows(n, nr, r, plane=36)
            S = gen.make("C2", N=6, row_begin=b, row_end=e)
            G = P.A.to_scipy()[b:e]
            assert (abs(S.A.to_scipy() - G)).max() == 0


# --------------------------------------------------------------- dots, norms
def test_dot_vs_fsum(orc):
    rng = np.random.default_rng(1)
    for n in (0, 1, 4095, 4096, 4097, 100_003):
        x = rng.standard_normal(n)
        y = rng.standard_normal(n)
        exact = math.fsum(x * y) if n else 0.0  # products are exact to 1/2 ulp
        d = orc.dot(x, y)
        scale = max(np.linalg.norm(x) * np.linalg.norm(y), 1e-300)
        assert abs(d - exact) <= 1e-15 * scale + 1e-300


def test_frobenius_examples(orc):
    assert orc.frobenius(_csr_of_dense(GOLD["frobenius_2x2"]["A"])) ** 2 == pytest.approx(10, rel=1e-15)
    assert orc.frobenius(sp.identity(3, format="csr")) ** 2 == pytest.approx(3, rel=1e-15)


def test_jacobi_diag_examples(orc, gen):
    A = sp.diags([np.arange(1.0, 6.0)], [0]).tocsr()
    assert np.allclose(orc.jacobi_diag(A), GOLD["jacobi_diag"]["M"], rtol=1e-15, atol=0)
    M = orc.jacobi_diag(gen.make("C1").A)
    assert np.all(M == 0.5)
    # floor case: zero diagonal entry floored by 1e-8 * max |A_jj|
    A = sp.csr_matrix(np.array([[0.0, 1.0], [1.0, 4.0]]))
    M = orc.jacobi_diag(A)
    assert M[0] == pytest.approx(1.0 / (1e-8 * 4.0)) and M[1] == 0.25
    # pencil: 1/|A_ii - sigma B_ii|
    P = gen.make("C4", N=4)
    Ad = P.A.to_scipy().diagonal()
    Bd = P.B.to_scipy().diagonal()
    M = orc.jacobi_diag(P.A, P.B, sigma=0.3)
    assert np.allclose(M, 1.0 / np.abs(Ad - 0.3 * Bd), rtol=1e-15)


# ------------------------------------------------------------- small eig (S6)
def test_sym_eig_spec_examples(orc):
    th, Y = orc.sym_eig(np.array(GOLD["eig_diag"]["T"], float))
    assert np.array_equal(th, [1, 2, 3])
    assert np.array_equal(Y, np.array(GOLD["eig_diag"]["Y"], float))
    th, Y = orc.sym_eig(np.array(GOLD["eig_2x2"]["T"], float))
    assert np.allclose(th, [1, 3], atol=1e-15)
    assert np.allclose(Y * np.sqrt(2), np.array(GOLD["eig_2x2"]["Y_scaled_by_sqrt2"], float), atol=1e-15)


@pytest.mark.parametrize("k", [1, 2, 5, 20, 48])
def test_sym_eig_vs_lapack(orc, k):
    rng = np.random.default_rng(k)
    R = rng.standard_normal((k, k))
    T = R + R.T
    th, Y = orc.sym_eig(T)
    ref = np.linalg.eigh(T)[0]
    nT = np.linalg.norm(T, 2)
    assert np.max(np.abs(th - ref)) <= 1e-13 * nT
    assert np.all(np.diff(th) >= 0)
    assert np.max(np.abs(Y.T @ Y - np.eye(k))) <= 1e-13
    assert np.max(np.abs(T @ Y - Y * th)) <= 1e-13 * nT
    for c in range(k):  # sign rule: largest-magnitude entry positive
        assert Y[np.argmax(np.abs(Y[:, c])), c] > 0


def test_sym_eig_degenerate_and_graded(orc):
    # exact multiplicity (C3-like) and tiny eigenvalues next to O(1) ones (C1-like T)
    rng = np.random.default_rng(7)
    Q, _ = np.linalg.qr(rng.standard_normal((12, 12)))
    lam = np.array([1e-5, 1e-5, 1e-5, 3e-5, 2.0, 2.0, 3.5, 3.9, 1.0, 0.5, 0.25, 4.0])
    T = (Q * lam) @ Q.T
    T = 0.5 * (T + T.T)
    th, Y = orc.sym_eig(T)
    assert np.max(np.abs(th - np.sort(lam))) <= 1e-14 * 4
    assert np.max(np.abs(T @ Y - Y * th)) <= 1e-14 * 4 * 4


# ---------------------------------------------------------------- CGS2 (S4)
def test_cgs2_spec_examples(orc):
    g = GOLD["orth_exact_projection"]
    w, h, beta, brk, _ = orc.cgs2(np.array(g["V"], float), g["w"])
    assert not brk and beta == pytest.approx(1.0) and np.allclose(w, g["w_out"], atol=1e-16)
    g = GOLD["orth_already"]
    w, h, beta, brk, _ = orc.cgs2(np.array(g["V"], float), g["w"])
    assert not brk and beta == 1.0 and np.array_equal(w, g["w_out"])


def test_cgs2_dependent_breaks_down(orc):
    rng = np.random.default_rng(3)
    V, _ = np.linalg.qr(rng.standard_normal((50, 6)))
    w, h, beta, brk, _ = orc.cgs2(V, V @ rng.standard_normal(6))
    assert brk


def test_cgs2_B_orthogonality(orc, gen):
    rng = np.random.default_rng(4)
    n = 100
    B = (gen.make("C1", N=n).A.to_scipy() + 2 * sp.identity(n)).tocsr()
    # B-orthonormal V by dense Cholesky-QR (independent of the oracle)
    X = rng.standard_normal((n, 6))
    L = np.linalg.cholesky(X.T @ (B @ X))
    V = np.linalg.solve(L, X.T).T
    assert np.max(np.abs(V.T @ (B @ V) - np.eye(6))) < 1e-12
    w0 = rng.standard_normal(n)
    w, h, beta, brk, passes = orc.cgs2(V, w0, B)
    assert not brk and passes >= 2
    assert np.max(np.abs(V.T @ (B @ w))) <= 1e-12 * np.sqrt(w0 @ (B @ w0))
    assert beta == pytest.approx(np.sqrt(w @ (B @ w)), rel=1e-14)
    # w_in = w_out + V h exactly in exact arithmetic
    assert np.max(np.abs(w + V @ h - w0)) <= 1e-13 * np.max(np.abs(w0))
