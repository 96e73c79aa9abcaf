"""Kernel-level parity: each device kernel, called through the C ABI
(include/trplk_kernels.h), against the oracle's primitive on the same seeded
inputs (normwise <= 1e-12 for vectors, |d - d_orc| <=
1e-12 ||u|| ||v|| for dots).  Sizes span several CTAs/tiles and a ragged tail."""
import numpy as np
import pytest

from gpu_util import b_orthonormal_block, need_gpu, normwise, to_dev

pytestmark = pytest.mark.gpu

# (config, grid N): 19^3 = 6859 and 9^3 = 729 rows leave ragged 32-row slices; C1 n = 1000
CASES = [("C2", 19), ("C4", 9), ("C1", None), ("C2", 40)]


@pytest.fixture(scope="module")
def problems(gen):
    return {f"{c}-{N}": gen.make(c, N=N) for c, N in CASES}


def _ctx(trplk, P, fmt="auto"):
    """fmt 'sell' forces the SELL-32 device format (TRPLK_FORCE_SELL); stencils pick DIA."""
    import os
    if fmt == "sell":
        os.environ["TRPLK_FORCE_SELL"] = "1"
    try:
        return trplk.trplk_create(P.A, P.B)
    finally:
        os.environ.pop("TRPLK_FORCE_SELL", None)


def _random_sym(n, density, seed):
    """General symmetric sparse matrix (many diagonals -> SELL-32) with a dominant diagonal."""
    import scipy.sparse as sp
    R = sp.random(n, n, density=density, random_state=seed, format="csr")
    A = (R + R.T + sp.diags(np.full(n, 4.0))).tocsr()
    A.sort_indices()
    return A


def test_spmv_and_step1_general_sparse(orc):
    """Non-stencil matrix: SELL-32 path, ragged rows of very different lengths."""
    torch, trplk = need_gpu()
    from types import SimpleNamespace
    n = 3001
    A = _random_sym(n, 0.01, 3)
    P = SimpleNamespace(A=A, B=None)
    ctx = trplk.trplk_create(A, n_global=n)
    rng = np.random.default_rng(0)
    x = rng.standard_normal(n)
    y = torch.zeros(n, dtype=torch.float64, device="cuda")
    trplk.trplk_k_spmv(ctx, 0, to_dev(torch, x), y)
    assert normwise(y.cpu().numpy(), orc.spmv(A, x)) <= 1e-13
    k = 12
    U = b_orthonormal_block(orc, n, k, None, seed=4)
    Ud = to_dev(torch, U, ctx.ld)
    w = torch.zeros(ctx.ld, dtype=torch.float64, device="cuda")
    tcol, h1, wn = trplk.trplk_k_step1(ctx, Ud, ctx.ld, k, Ud[k - 1], 0.3, w)
    z = orc.spmv(A, U[:, k - 1])
    w_o = orc.jacobi_diag(A) * (z - 0.3 * U[:, k - 1])
    assert normwise(w.cpu().numpy()[:n], w_o) <= 1e-12
    assert np.all(np.abs(tcol - U.T @ z) <= 1e-12 * np.linalg.norm(z))
    assert np.all(np.abs(h1 - U.T @ w_o) <= 1e-12 * np.linalg.norm(w_o))
    del P


@pytest.mark.parametrize("case", [f"{c}-{N}" for c, N in CASES])
def test_spmv_sell_format(orc, problems, case):
    torch, trplk = need_gpu()
    P = problems[case]
    ctx = _ctx(trplk, P, "sell")
    n = P.A.n
    x = np.random.default_rng(5).standard_normal(n)
    y = torch.zeros(n, dtype=torch.float64, device="cuda")
    trplk.trplk_k_spmv(ctx, 0, to_dev(torch, x), y)
    assert normwise(y.cpu().numpy(), orc.spmv(P.A, x)) <= 1e-13
    r = torch.zeros(ctx.ld, dtype=torch.float64, device="cuda")
    u = torch.zeros(ctx.ld, dtype=torch.float64, device="cuda")
    trplk.trplk_k_residual(ctx, to_dev(torch, x, ctx.ld), 0.25, r, u)
    Bx = x if P.B is None else orc.spmv(P.B, x)
    r_o = orc.spmv(P.A, x) - 0.25 * Bx
    assert normwise(r.cpu().numpy()[:n], r_o) <= 1e-13
    assert normwise(u.cpu().numpy()[:n], orc.jacobi_diag(P.A, P.B) * r_o) <= 1e-13


@pytest.mark.parametrize("case", [f"{c}-{N}" for c, N in CASES])
def test_spmv_A_and_B(orc, problems, case):
    torch, trplk = need_gpu()
    P = problems[case]
    ctx = _ctx(trplk, P)
    n = P.A.n
    rng = np.random.default_rng(1)
    x = rng.standard_normal(n)
    y = torch.zeros(n, dtype=torch.float64, device="cuda")
    trplk.trplk_k_spmv(ctx, 0, to_dev(torch, x), y)
    assert normwise(y.cpu().numpy(), orc.spmv(P.A, x)) <= 1e-13
    if P.B is not None:
        trplk.trplk_k_spmv(ctx, 1, to_dev(torch, x), y)
        assert normwise(y.cpu().numpy(), orc.spmv(P.B, x)) <= 1e-13


@pytest.mark.parametrize("case", [f"{c}-{N}" for c, N in CASES])
@pytest.mark.parametrize("k", [1, 7, 20, 48])
def test_step1_fused_spmv_precond_dots(orc, problems, case, k):
    """K1: z = A g, T(1:k,k) = U^T z, w = M (z - rho B g), h1 = U^T B w, ||w||_B^2."""
    torch, trplk = need_gpu()
    P = problems[case]
    n = P.A.n
    if k >= n:
        pytest.skip("k >= n")
    ctx = _ctx(trplk, P)
    U = b_orthonormal_block(orc, n, k, P.B, seed=k)
    g = U[:, k - 1]
    rho = 0.5
    Ud = to_dev(torch, U, ctx.ld)
    w = torch.zeros(ctx.ld, dtype=torch.float64, device="cuda")
    tcol, h1, wn = trplk.trplk_k_step1(ctx, Ud, ctx.ld, k, Ud[k - 1], rho, w)
    # oracle
    z = orc.spmv(P.A, g)
    s = g if P.B is None else orc.spmv(P.B, g)
    M = orc.jacobi_diag(P.A, P.B)
    w_o = M * (z - rho * s)
    Bw = w_o if P.B is None else orc.spmv(P.B, w_o)
    t_o = np.array([orc.dot(U[:, i], z) for i in range(k)])
    h_o = np.array([orc.dot(U[:, i], Bw) for i in range(k)])
    assert normwise(w.cpu().numpy()[:n], w_o) <= 1e-12
    nz, nBw = np.linalg.norm(z), np.linalg.norm(Bw)
    un = np.linalg.norm(U, axis=0)
    assert np.all(np.abs(tcol - t_o) <= 1e-12 * un * nz)
    assert np.all(np.abs(h1 - h_o) <= 1e-12 * un * nBw)
    assert abs(wn - orc.dot(w_o, Bw)) <= 1e-12 * np.linalg.norm(w_o) * nBw


@pytest.mark.parametrize("case", [f"{c}-{N}" for c, N in CASES])
@pytest.mark.parametrize("k", [0, 5, 33])
def test_cgs2_B_inner_product(orc, problems, case, k):
    torch, trplk = need_gpu()
    P = problems[case]
    n = P.A.n
    ctx = _ctx(trplk, P)
    U = b_orthonormal_block(orc, n, max(k, 1), P.B, seed=11)[:, :k]
    rng = np.random.default_rng(k + 3)
    w0 = rng.standard_normal(n)
    Ud = to_dev(torch, U if k else np.zeros((n, 1)), ctx.ld)
    out = torch.zeros(ctx.ld, dtype=torch.float64, device="cuda")
    h, beta, brk, passes = trplk.trplk_k_cgs2(ctx, Ud, ctx.ld, k, to_dev(torch, w0, ctx.ld), out)
    w_o, h_o, beta_o, brk_o, passes_o = orc.cgs2(U if k else np.zeros((n, 0)), w0, P.B)
    assert brk == brk_o is False and passes == passes_o
    assert abs(beta - beta_o) <= 1e-12 * beta_o
    assert normwise(out.cpu().numpy()[:n], w_o / beta_o) <= 1e-12
    assert np.all(np.abs(h - h_o) <= 1e-12 * np.linalg.norm(w0))
    # dependent vector: both break down (R16)
    if k:
        wd = U @ rng.standard_normal(k)
        _, _, brk, _ = trplk.trplk_k_cgs2(ctx, Ud, ctx.ld, k, to_dev(torch, wd, ctx.ld), out)
        assert brk and orc.cgs2(U, wd, P.B)[3]


@pytest.mark.parametrize("case", ["C2-19", "C4-9"])
@pytest.mark.parametrize("k", [5, 33])
def test_cgs2_forced_third_pass(orc, problems, case, k):
    """Reading R3's third pass, forced (trplk_set_debug): B = I runs it inside the cooperatively
    launched FINAL kernel, B != I through the gated pass-3 launches.  A third projection of a
    vector already B-orthogonal to U changes it only at rounding level, so the result must still
    equal the oracle's two-pass CGS2 (normwise 1e-12) and report 3 passes."""
    torch, trplk = need_gpu()
    P = problems[case]
    n = P.A.n
    ctx = _ctx(trplk, P)
    trplk.trplk_set_debug(ctx, 1)
    U = b_orthonormal_block(orc, n, k, P.B, seed=13)
    w0 = np.random.default_rng(k + 7).standard_normal(n)
    out = torch.zeros(ctx.ld, dtype=torch.float64, device="cuda")
    h, beta, brk, passes = trplk.trplk_k_cgs2(ctx, to_dev(torch, U, ctx.ld), ctx.ld, k, to_dev(torch, w0, ctx.ld),
                                              out)
    w_o, h_o, beta_o, brk_o, passes_o = orc.cgs2(U, w0, P.B)
    assert passes == 3 and not brk and not brk_o
    assert abs(beta - beta_o) <= 1e-12 * beta_o
    assert normwise(out.cpu().numpy()[:n], w_o / beta_o) <= 1e-12
    assert np.all(np.abs(h - h_o) <= 1e-12 * np.linalg.norm(w0))
    trplk.trplk_set_debug(ctx, 0)


@pytest.mark.parametrize("ncol", [1, 5, 8, 10, 20, 24])
@pytest.mark.parametrize("k", [1, 6, 30, 64])
def test_rotate_dmma(orc, problems, ncol, k):
    """K5: X = U Y on fp64 DMMA vs the oracle's triple loop."""
    torch, trplk = need_gpu()
    P = problems["C2-19"]
    n = P.A.n
    ctx = _ctx(trplk, P)
    rng = np.random.default_rng(ncol * 100 + k)
    U = rng.standard_normal((n, k))
    Y = rng.standard_normal((k, ncol))
    X = torch.zeros((ncol, ctx.ld), dtype=torch.float64, device="cuda")
    trplk.trplk_k_rotate(ctx, to_dev(torch, U, ctx.ld), ctx.ld, k, Y, ncol, X, ctx.ld)
    Xo = orc.rotate(U, Y)
    assert normwise(X.cpu().numpy()[:, :n].T, Xo) <= 1e-13


@pytest.mark.parametrize("k", [1, 2, 5, 20, 31, 48, 64])
def test_sym_eig_one_cta_jacobi(orc, problems, k):
    torch, trplk = need_gpu()
    ctx = _ctx(trplk, problems["C1-None"])
    rng = np.random.default_rng(k)
    R = rng.standard_normal((k, k))
    T = R + R.T
    th, Y = trplk.trplk_k_sym_eig(ctx, T)
    th_o, Y_o = orc.sym_eig(T)
    nT = np.linalg.norm(T, 2)
    assert np.max(np.abs(th - th_o)) <= 1e-13 * nT
    assert np.max(np.abs(Y.T @ Y - np.eye(k))) <= 1e-13
    assert np.max(np.abs(T @ Y - Y * th)) <= 1e-13 * nT
    gaps = np.min(np.abs(np.subtract.outer(th_o, th_o)) + np.eye(k) * 1e9, axis=1)
    for c in range(k):  # unique eigenvectors (distinct eigenvalues + sign rule) agree
        assert np.max(np.abs(Y[:, c] - Y_o[:, c])) <= 1e-13 * nT / gaps[c] + 1e-14


def test_sym_eig_degenerate_graded(orc, problems):
    torch, trplk = need_gpu()
    ctx = _ctx(trplk, problems["C1-None"])
    rng = np.random.default_rng(9)
    Q, _ = np.linalg.qr(rng.standard_normal((24, 24)))
    lam = np.r_[[1e-5] * 3, 3e-5, [2.0] * 6, np.linspace(0.1, 4, 14)]
    T = (Q * lam) @ Q.T
    T = 0.5 * (T + T.T)
    th, Y = trplk.trplk_k_sym_eig(ctx, T)
    assert np.max(np.abs(th - np.sort(lam))) <= 1e-14 * 8
    assert np.max(np.abs(T @ Y - Y * th)) <= 1e-14 * 40


@pytest.mark.parametrize("case", [f"{c}-{N}" for c, N in CASES])
def test_residual_and_seed(orc, problems, case):
    torch, trplk = need_gpu()
    P = problems[case]
    n = P.A.n
    ctx = _ctx(trplk, P)
    rng = np.random.default_rng(2)
    x = rng.standard_normal(n)
    theta = 0.37
    r = torch.zeros(ctx.ld, dtype=torch.float64, device="cuda")
    u = torch.zeros(ctx.ld, dtype=torch.float64, device="cuda")
    n2 = trplk.trplk_k_residual(ctx, to_dev(torch, x, ctx.ld), theta, r, u)
    Bx = x if P.B is None else orc.spmv(P.B, x)
    r_o = orc.spmv(P.A, x) - theta * Bx
    M = orc.jacobi_diag(P.A, P.B)
    assert normwise(r.cpu().numpy()[:n], r_o) <= 1e-13
    assert normwise(u.cpu().numpy()[:n], M * r_o) <= 1e-13
    assert abs(n2 - orc.dot(r_o, r_o)) <= 1e-12 * orc.dot(r_o, r_o)


def test_random_start_block_bit_exact(orc, problems):
    """Counter-based generator (R13): device draws equal the oracle's bit for bit."""
    torch, trplk = need_gpu()
    P = problems["C2-19"]
    n = P.A.n
    ctx = _ctx(trplk, P)
    x = torch.zeros(n, dtype=torch.float64, device="cuda")
    for stream, col in ((0, 0), (0, 7), (2, 3)):
        trplk.trplk_k_random(ctx, 12, stream, col, x)
        ref = np.array([orc.u01(12, stream, col * n + i) for i in range(n)])
        assert np.array_equal(x.cpu().numpy(), ref)


@pytest.mark.parametrize("diac", ["1", "0"])
@pytest.mark.parametrize("k", [8, 13, 16])
def test_step1_pipe_full_slab(orc, gen, k, diac):
    """The K1 that C5 runs for k <= 16 on slabs of >= 2^24 rows: the thread-per-row k_step1_lean
    with the DIA-C decode (default), or k_step1_pipe when the matrix has no presence bits
    (TRPLK_DIAC=0) -- at a size that selects them: 257^3 = 16,974,593 rows (ragged last 32-row
    tile), C5's matrix shape (7-pt + diag(d), d~U[0,10)).  Every output against the oracle's SpMV
    and blocked dots over all rows: w normwise <= 1e-12, dots <= 1e-12 ||u|| ||v||."""
    import os
    torch, trplk = need_gpu()
    P = gen.make("C5", N=257)
    n = P.A.n
    assert n >= 1 << 24
    os.environ["TRPLK_DIAC"] = diac
    try:
        ctx = trplk.trplk_create(P.A, P.B)
    finally:
        os.environ.pop("TRPLK_DIAC", None)
    rng = np.random.default_rng(100 + k)
    U = np.asfortranarray(rng.standard_normal((n, k)) / np.sqrt(n))
    g = U[:, k - 1]
    rho = 2.75
    Ud = to_dev(torch, U, ctx.ld)
    w = torch.zeros(ctx.ld, dtype=torch.float64, device="cuda")
    tcol, h1, wn = trplk.trplk_k_step1(ctx, Ud, ctx.ld, k, Ud[k - 1], rho, w)
    z = orc.spmv(P.A, g)
    w_o = orc.jacobi_diag(P.A) * (z - rho * g)
    assert normwise(w.cpu().numpy()[:n], w_o) <= 1e-12
    un, nz, nw = np.linalg.norm(U, axis=0), np.linalg.norm(z), np.linalg.norm(w_o)
    t_o = np.array([orc.dot(U[:, i], z) for i in range(k)])
    h_o = np.array([orc.dot(U[:, i], w_o) for i in range(k)])
    assert np.all(np.abs(tcol - t_o) <= 1e-12 * un * nz)
    assert np.all(np.abs(h1 - h_o) <= 1e-12 * un * nw)
    assert abs(wn - orc.dot(w_o, w_o)) <= 1e-12 * nw * nw
    ctx.close()


@pytest.mark.parametrize("case", ["C2-19", "C2-40", "C1-None"])
@pytest.mark.parametrize("k,c", [(1, 1), (7, 2), (22, 2), (45, 3), (64, 8), (30, 5)])
def test_block_kernels_gram_upd_spmm(orc, problems, case, k, c):
    """The block +K kernels (block.cuh) against the oracle's primitives: GRAM U^T Y and Y^T Y,
    UPD Y' = Y R^-1 - U H with its U^T Y', Y'^T Y', SPMM U^T (A Y) -- dots within
    1e-12 ||u|| ||v||, vectors normwise 1e-12; ragged row tails and every DMMA chunk width."""
    torch, trplk = need_gpu()
    P = problems[case]
    n = P.A.n
    if k + c > n:
        pytest.skip("block wider than the problem")
    ctx = _ctx(trplk, P)
    rng = np.random.default_rng(1000 + 10 * k + c)
    U = rng.standard_normal((n, k)) / np.sqrt(n)
    Y = rng.standard_normal((n, c))
    Ud, Yd = to_dev(torch, U, ctx.ld), to_dev(torch, Y, ctx.ld)
    un, yn = np.linalg.norm(U, axis=0), np.linalg.norm(Y, axis=0)
    # GRAM
    HV, G = trplk.trplk_k_block(ctx, 0, Ud, ctx.ld, k, Yd, ctx.ld, c)
    HVo = np.array([[orc.dot(U[:, i], Y[:, j]) for j in range(c)] for i in range(k)])
    Go = np.array([[orc.dot(Y[:, i], Y[:, j]) for j in range(c)] for i in range(c)])
    assert np.all(np.abs(HV - HVo) <= 1e-12 * np.outer(un, yn))
    assert np.all(np.abs(G - Go) <= 1e-12 * np.outer(yn, yn))
    # UPD with an upper-triangular R^-1 and coefficients H
    R = np.triu(rng.standard_normal((c, c))) + 3 * np.eye(c)
    H = rng.standard_normal((k, c))
    Yo = torch.zeros((c, ctx.ld), dtype=torch.float64, device="cuda")
    HV, G = trplk.trplk_k_block(ctx, 1, Ud, ctx.ld, k, Yd, ctx.ld, c, Rinv=R, H=H, Yout=Yo, ldyo=ctx.ld)
    Q = Y @ R  # Q = Y Rinv with Rinv := R here
    Yp = Q - U @ H
    Ypg = Yo.cpu().numpy()[:, :n].T
    assert normwise(Ypg, Yp) <= 1e-12
    ypn = np.linalg.norm(Yp, axis=0)
    HVo = np.array([[orc.dot(U[:, i], Yp[:, j]) for j in range(c)] for i in range(k)])
    Go = np.array([[orc.dot(Yp[:, i], Yp[:, j]) for j in range(c)] for i in range(c)])
    assert np.all(np.abs(HV - HVo) <= 1e-11 * np.outer(un, ypn))
    assert np.all(np.abs(G - Go) <= 1e-11 * np.outer(ypn, ypn))
    # SPMM
    HV, _ = trplk.trplk_k_block(ctx, 2, Ud, ctx.ld, k, Yd, ctx.ld, c)
    Z = np.stack([orc.spmv(P.A, Y[:, j]) for j in range(c)], axis=1)
    HVo = np.array([[orc.dot(U[:, i], Z[:, j]) for j in range(c)] for i in range(k)])
    assert np.all(np.abs(HV - HVo) <= 1e-12 * np.outer(un, np.linalg.norm(Z, axis=0)))
    ctx.close()


@pytest.mark.parametrize("ncol,k", [(20, 48), (24, 40), (8, 32), (10, 24), (3, 16)])
def test_rotate_dmma_pipelined(orc, gen, ncol, k):
    """K5 with several 32-row tiles per warp (the cp.async double-buffered slab: the next tile
    streams in while the current one is in the DMMA) and a ragged tail (65^3 = 274,625 rows,
    one row past a tile boundary), against the oracle's triple loop."""
    torch, trplk = need_gpu()
    P = gen.make("C2", N=65)
    n = P.A.n
    assert n % 32 == 1
    ctx = _ctx(trplk, P)
    rng = np.random.default_rng(ncol * 1000 + k)
    U = rng.standard_normal((n, k))
    Y = rng.standard_normal((k, ncol))
    X = torch.zeros((ncol, ctx.ld), dtype=torch.float64, device="cuda")
    trplk.trplk_k_rotate(ctx, to_dev(torch, U, ctx.ld), ctx.ld, k, Y, ncol, X, ctx.ld)
    Xo = orc.rotate(U, Y)
    assert normwise(X.cpu().numpy()[:, :n].T, Xo) <= 1e-13
