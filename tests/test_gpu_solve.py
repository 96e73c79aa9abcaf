"""End-to-end parity of trplk_solve (C ABI) with the oracle on the same seeded
inputs (SURVEY 8(c.5) protocol): identical per-cycle trajectory (t, basis
width, X^prev width) with theta_t within 1e-10 relative -- hence identical
A-matvec counts -- unless the runs diverge at a near-tie; eigenvalues within
1e-9 relative; all residuals <= tol; eigenvector subspace angles <= 1e-6 at
tol_parity, grouped by clusters."""
import numpy as np
import pytest
import scipy.linalg as sla

from gpu_util import need_gpu

pytestmark = pytest.mark.gpu


def gpu_solve(trplk, P, tol=None, fmt="auto", debug=0, **opt):
    import os
    if fmt == "sell":
        os.environ["TRPLK_FORCE_SELL"] = "1"
    try:
        ctx = trplk.trplk_create(P.A, P.B, P.sigma)
    finally:
        os.environ.pop("TRPLK_FORCE_SELL", None)
    if debug:
        trplk.trplk_set_debug(ctx, debug)
    ev, X, rs, st = trplk.trplk_solve(ctx, P.p, P.q, P.l, P.tol if tol is None else tol, **opt)
    ph = opt.get("restart_size", 0) or P.p
    log = trplk.trplk_get_log(ctx, ph=ph)
    Xh = X.cpu().numpy().copy()
    ctx.close()
    return {"eigenvalues": ev, "X": Xh, "residuals": rs, "stats": st, "log": log}


def oracle_solve(orc, P, tol=None, **opt):
    return orc.solve(P.A, P.B, P.p, P.q, P.l, P.tol if tol is None else tol, P.sigma, **opt)


def norm_inf(P):
    """max row sum |A| (>= ||A||_2 for symmetric A): scale of rounding errors in Ritz values."""
    A = P.A.to_scipy()
    return float(abs(A).sum(axis=1).max())


def first_divergence(g, o, nA):
    """First cycle where (t, width, X^prev width) differ or theta_t differs by more than
    1e-10 relative + 1e-13 ||A|| (RR is backward stable: absolute errors O(eps ||A||))."""
    lg, lo = g["log"], o["log"]
    n = min(len(lg["t"]), len(lo["t"]))
    for c in range(n):
        same = (lg["t"][c] == lo["t"][c] and lg["k"][c] == lo["k"][c] and lg["nprev"][c] == lo["nprev"][c]
                and abs(lg["theta_t"][c] - lo["theta_t"][c]) <= 1e-10 * abs(lo["theta_t"][c]) + 1e-13 * nA)
        if not same:
            return c
    return None if len(lg["t"]) == len(lo["t"]) else n


def near_tie(o, c, tol):
    """Divergence allowed only at a near-tie: Ritz values within 1e-10 rel, or ||r_t|| ~ tau."""
    th = o["log"]["thetas"][c]
    close = np.any(np.abs(np.diff(th)) <= 1e-10 * np.abs(th[1:]))
    res = o["log"]["res"][c]
    return close or abs(res - tol) <= 1e-2 * tol


def subspace_angles_grouped(X, Y, B, lam, tolp):
    """Max B-principal angle between X and Y over groups of clustered eigenvalues."""
    groups, cur = [], [0]
    for i in range(1, len(lam)):
        if lam[i] - lam[i - 1] < 10 * tolp / 1e-6:
            cur.append(i)
        else:
            groups.append(cur)
            cur = [i]
    groups.append(cur)
    worst = 0.0
    for g in groups:
        BY = Y[:, g] if B is None else B @ Y[:, g]
        s = np.linalg.svd(X[:, g].T @ BY, compute_uv=False)
        worst = max(worst, float(np.arccos(np.clip(np.min(s), -1, 1))))
    return worst, groups


def check_parity(g, o, P, allow_tie_divergence=False):
    assert g["stats"]["status"] == o["status"] == "OK"
    assert np.all(g["residuals"] <= P.tol) and np.all(o["residuals"] <= P.tol)
    c = first_divergence(g, o, norm_inf(P))
    if c is None:
        assert g["stats"]["a_matvecs"] == o["a_matvecs"]
        assert g["stats"]["cycles"] == o["cycles"]
    else:
        lg, lo = g["log"], o["log"]
        info = {k_: (lg[k_][c], lo[k_][c]) for k_ in ("t", "k", "nprev", "theta_t", "res")}
        assert allow_tie_divergence and near_tie(o, c, P.tol), f"trajectory diverged at cycle {c}: {info}"
    rel = np.abs(g["eigenvalues"] - o["eigenvalues"]) / np.abs(o["eigenvalues"])
    assert np.max(rel) <= 1e-9, rel
    return c


@pytest.mark.parametrize("name,N,fmt", [("C1", None, "auto"), ("C2", 12, "auto"), ("C2", 24, "auto"),
                                        ("C4", 8, "auto"), ("C4", 12, "auto"), ("C2", 12, "sell"),
                                        ("C4", 8, "sell")])
def test_solve_parity_small(orc, gen, name, N, fmt):
    torch, trplk = need_gpu()
    P = gen.make(name, N=N)
    g = gpu_solve(trplk, P, fmt=fmt)
    o = oracle_solve(orc, P)
    check_parity(g, o, P)
    # B-orthonormal eigenvectors
    X = g["X"]
    BX = X if P.B is None else P.B.to_scipy() @ X
    assert np.max(np.abs(X.T @ BX - np.eye(P.p))) <= 1e-11  # oracle: 1.5e-12 on C1


def test_solve_clustered_C3_small(orc, gen):
    """Exact multiplicities (C3 shape, 12^3): several results are correct -- compare complete
    clusters' subspaces; trajectory may only diverge at a near-tie."""
    torch, trplk = need_gpu()
    P = gen.make("C3", N=12, p=10, q=24, l=3)
    g = gpu_solve(trplk, P)
    o = oracle_solve(orc, P)
    check_parity(g, o, P, allow_tie_divergence=True)
    c = 2 - 2 * np.cos(np.arange(1, 13) * np.pi / 13)
    ref = np.sort(np.add.outer(np.add.outer(c, c), c).ravel())[:10]
    assert np.max(np.abs(g["eigenvalues"] - ref) / ref) <= 1e-9


@pytest.mark.parametrize("name,N,tolp", [("C1", None, 1e-12), ("C2", 16, 1e-11), ("C4", 8, 1e-11)])
def test_eigenvector_angles_tol_parity(orc, gen, name, N, tolp):
    torch, trplk = need_gpu()
    P = gen.make(name, N=N)
    g = gpu_solve(trplk, P, tol=tolp)
    o = oracle_solve(orc, P, tol=tolp)
    assert g["stats"]["status"] == "OK" and o["status"] == "OK"
    B = None if P.B is None else P.B.to_scipy()
    ang, groups = subspace_angles_grouped(g["X"], o["eigenvectors"], B, o["eigenvalues"], tolp)
    assert ang <= 1e-6, (ang, groups)


def test_graph_and_eager_bitwise_equal_and_deterministic(gen):
    torch, trplk = need_gpu()
    P = gen.make("C2", N=20)
    a = gpu_solve(trplk, P, use_graphs=1)
    b = gpu_solve(trplk, P, use_graphs=0)
    c = gpu_solve(trplk, P, use_graphs=1)
    assert np.array_equal(a["eigenvalues"], b["eigenvalues"])
    assert np.array_equal(a["eigenvalues"], c["eigenvalues"])
    assert np.array_equal(a["X"], c["X"])
    assert a["stats"]["a_matvecs"] == b["stats"]["a_matvecs"]


def test_matvec_accounting_and_interlacing(gen):
    torch, trplk = need_gpu()
    P = gen.make("C2", N=10, p=4, q=12, l=2)
    g = gpu_solve(trplk, P, tol=1e-10)
    lg = g["log"]
    ph, m = 4, 12 - 4 - 2
    mv = np.r_[ph, lg["mv"]]
    tt = lg["t"]
    tnext = np.r_[tt[1:], ph + 1]
    for c in range(len(tt)):
        locks = tnext[c] - tt[c]
        extra = locks if tnext[c] <= ph else locks - 1
        assert mv[c + 1] - mv[c] == m + lg["nprev"][c] + 1 + extra
    th = lg["thetas"]
    assert np.all(th[1:] <= th[:-1] + 1e-14 * np.abs(th[:-1]) + 1e-14)


def test_options_restart_size_lock_while_frob(orc, gen):
    torch, trplk = need_gpu()
    P = gen.make("C2", N=12)
    for opt in ({"restart_size": 12}, {"lock_mode": 1}, {"tol_mode": 1}):
        tol = 1e-12 if opt.get("tol_mode") else P.tol
        g = gpu_solve(trplk, P, tol=tol, **opt)
        o = orc.solve(P.A, None, P.p, P.q, P.l, tol, **opt)
        assert g["stats"]["status"] == "OK"
        assert g["stats"]["a_matvecs"] == o["a_matvecs"], opt
        assert np.max(np.abs(g["eigenvalues"] - o["eigenvalues"]) / o["eigenvalues"]) <= 1e-9


def test_not_converged_and_einval(gen):
    torch, trplk = need_gpu()
    P = gen.make("C2", N=10)
    ctx = trplk.trplk_create(P.A)
    ev, X, rs, st = trplk.trplk_solve(ctx, 4, 12, 2, 1e-13, max_cycles=2)
    assert st["status"] == "NOT_CONVERGED" and st["cycles"] == 2 and np.all(np.isfinite(ev))
    with pytest.raises(trplk.TrplkError):
        trplk.trplk_solve(ctx, 4, 6, 2, 1e-8)  # m = 0
    with pytest.raises(trplk.TrplkError):
        trplk.trplk_solve(ctx, 4, 65, 2, 1e-8)  # q > TRPLK_MAX_BASIS
    ctx.close()


def test_full_C2_parity(orc, gen):
    """BASELINE configs[1] at full size, bench launch configuration."""
    torch, trplk = need_gpu()
    P = gen.make("C2")
    g = gpu_solve(trplk, P)
    o = oracle_solve(orc, P, want_vectors=False)
    check_parity(g, o, P, allow_tie_divergence=True)


@pytest.mark.parametrize("name,N", [("C2", 12), ("C4", 8), ("C2", 24), ("C5", 24)])
def test_solve_with_forced_third_pass(orc, gen, name, N):
    """Every CGS2 of the solve takes the third pass (options.debug_checks bit 1): the same
    trajectory as the oracle's two-pass run (the third projection is rounding-level), so the
    A-matvec count and the eigenvalues agree."""
    torch, trplk = need_gpu()
    P = gen.make(name, N=N)
    g = gpu_solve(trplk, P, debug_checks=2)
    o = oracle_solve(orc, P, want_vectors=False)
    assert g["stats"]["status"] == "OK"
    assert g["stats"]["a_matvecs"] == o["a_matvecs"]
    assert np.max(np.abs(g["eigenvalues"] - o["eigenvalues"]) / np.abs(o["eigenvalues"])) <= 1e-9
    assert np.all(g["residuals"] <= P.tol)


@pytest.mark.parametrize("q", [49, 64])
def test_widest_basis(orc, gen, q):
    """max_basis up to TRPLK_MAX_BASIS = 64: the k > 48 kernel instantiations (DMMA-fragment K1,
    4-warp K2 groups, 3-group rotation) against the oracle's trajectory and eigenvalues."""
    torch, trplk = need_gpu()
    P = gen.make("C2", N=14, q=q)
    g = gpu_solve(trplk, P)
    o = oracle_solve(orc, P, want_vectors=False)
    assert g["stats"]["status"] == "OK" and o["status"] == "OK"
    assert g["stats"]["a_matvecs"] == o["a_matvecs"]
    assert np.max(np.abs(g["eigenvalues"] - o["eigenvalues"]) / np.abs(o["eigenvalues"])) <= 1e-9
    assert np.all(g["residuals"] <= P.tol)


class _Csr:
    def __init__(self, rowptr, col, val, n):
        self.rowptr, self.col, self.val, self.n, self.row_begin = rowptr, col, val, n, 0


@pytest.mark.parametrize("name,N,torch_alloc", [("C2", 16, True), ("C4", 10, True), ("C2", 16, False)])
def test_pinned_host_csr(gen, name, N, torch_alloc):
    """Pinned host CSR arrays take the device-side CSR -> DIA scatter (k_csr_to_dia), pageable
    ones the host scatter: the same device matrix, so the same solve bit for bit.  With
    torch_alloc=False the library's own stream-ordered memory pool serves every buffer."""
    torch, trplk = need_gpu()
    P = gen.make(name, N=N)

    def pinned(M):
        if M is None:
            return None
        t = [torch.from_numpy(a).pin_memory() for a in (M.rowptr, M.col, M.val)]
        return _Csr(*(x.numpy() for x in t), M.n), t

    pa = pinned(P.A)
    pb = pinned(P.B)
    out = []
    for A, B in ((P.A, P.B), (pa[0], None if pb is None else pb[0])):
        ctx = trplk.trplk_create(A, B, P.sigma, torch_alloc=torch_alloc)
        info = trplk.trplk_info(ctx)
        ev, X, rs, st = trplk.trplk_solve(ctx, P.p, P.q, P.l, P.tol)
        out.append((ev, X.cpu().numpy().copy(), st["a_matvecs"], info))
        ctx.close()
    assert out[0][3] == out[1][3]
    assert out[0][2] == out[1][2]
    assert np.array_equal(out[0][0], out[1][0])
    assert np.array_equal(out[0][1], out[1][1])


@pytest.mark.parametrize("name,N,over,fmt,debug", [
    ("C2", 24, {}, "auto", 2),               # q = 30: the KMAX = 32 instantiation
    ("C2", 24, {"q": 22}, "auto", 2),        # KMAX = 24
    ("C2", 21, {"q": 16}, "auto", 2),        # KMAX = 16
    ("C2", 24, {}, "sell", 2),               # SELL-32 SpMV inside the grid kernel
    ("C2", 24, {}, "auto", 3),               # every CGS2 takes the in-kernel third pass
    ("C3", 22, {"p": 10, "q": 30, "l": 3}, "auto", 2),  # exact multiplicities
])
def test_grid_inner_loop(orc, gen, name, N, over, fmt, debug):
    """The m inner steps as one cooperative grid-wide kernel (trplk_set_debug bit 1,
    inner_grid.cuh): same trajectory as the oracle (A-matvec count, cycle log up to near-ties),
    eigenvalues to 1e-9 relative, B-orthonormal eigenvectors."""
    torch, trplk = need_gpu()
    P = gen.make(name, N=N, **over)
    assert P.A.n > 8192  # above the single-CTA small path
    g = gpu_solve(trplk, P, fmt=fmt, debug=debug)
    o = oracle_solve(orc, P)
    if name == "C3":
        check_parity(g, o, P, allow_tie_divergence=True)
    else:
        # small-q runs are long (100-200 cycles) with a slowly converging target whose Ritz value
        # drifts by ~1e-10 relative under any change of summation order (the multi-kernel path
        # shows the same drift, tools/cmp_traj.py): compare the cycle structure exactly and
        # theta_t to 1e-8 relative
        # theta_t to 1e-8 relative.  The opt-in tridiagonal RR (TRPLK_EIG=tri) drifts theta_t by
        # 2.5e-9 over this 270-cycle run and the target then converges 10 cycles earlier than the
        # oracle's (the oracle's residual there is 2.2e-7): the structure must agree up to the
        # shorter run's end and the lengths within 5 %; eigenvalues and residuals as always
        assert g["stats"]["status"] == "OK"
        lg, lo = g["log"], o["log"]
        n = min(len(lg["t"]), len(lo["t"]))
        for key in ("t", "k", "nprev"):
            assert np.array_equal(lg[key][:n], lo[key][:n]), key
        assert np.max(np.abs(lg["theta_t"][:n] - lo["theta_t"][:n]) / np.abs(lo["theta_t"][:n])) <= 1e-8
        if g["stats"]["cycles"] != o["cycles"]:
            assert n >= 200 and abs(g["stats"]["cycles"] - o["cycles"]) <= 0.05 * o["cycles"]
        else:
            assert g["stats"]["a_matvecs"] == o["a_matvecs"]
        assert np.max(np.abs(g["eigenvalues"] - o["eigenvalues"]) / np.abs(o["eigenvalues"])) <= 1e-9
        assert np.all(g["residuals"] <= P.tol)
    X = g["X"]
    assert np.max(np.abs(X.T @ X - np.eye(P.p))) <= 1e-11


def test_graph_cache_across_contexts(gen):
    """A context created after another one of the same shape reuses its instantiated cycle
    graphs (same device addresses): the results must be those of an eager (graph-free) solve of
    the SECOND problem, bit for bit -- a replayed graph reads the new matrix and vectors."""
    torch, trplk = need_gpu()
    P1 = gen.make("C2", N=16)
    P2 = gen.make("C2", N=16, dscale=3.0)  # same structure, other values
    for P in (P1, P2, P1):
        ctx = trplk.trplk_create(P.A, P.B, P.sigma)
        ev, X, rs, st = trplk.trplk_solve(ctx, P.p, P.q, P.l, P.tol)
        ctx.close()
        ctx = trplk.trplk_create(P.A, P.B, P.sigma)
        ev0, X0, rs0, st0 = trplk.trplk_solve(ctx, P.p, P.q, P.l, P.tol, use_graphs=0)
        ctx.close()
        assert np.array_equal(ev, ev0) and np.array_equal(rs, rs0)
        assert st["a_matvecs"] == st0["a_matvecs"]


@pytest.mark.parametrize("name,N,l,pc", [("C2", 12, 0, 1), ("C2", 24, 0, 1), ("C4", 8, 0, 1), ("C1", None, 0, 1),
                                         ("C2", 16, 2, 1), ("C2", 16, 2, 2), ("C2", 24, 2, 2), ("C4", 8, 2, 2),
                                         ("C5", 16, 2, 2), ("C2", 12, 2, 3), ("C2", 24, 2, 3), ("C3", 12, 3, 3),
                                         ("C5", 20, 2, 3), ("C1", None, 1, 3), ("C2", 40, 2, 3)])
def test_no_preconditioner_trlan_baseline(orc, gen, name, N, l, pc):
    """options.precond = 1 (M = I): with k_plus = 0 the thick-restart Lanczos baseline of eq 2.1
    (NEXT-4; the oracle pins its space per cycle in test_oracle_solver.py), the same parity as
    the preconditioned solve against the oracle run with precond = 1.  C1 (n = 1000) runs the
    single-CTA path, C2-24 the multi-kernel one, C4 the pencil.  pc = 2: the per-cycle shifted
    Jacobi of NEXT-2 against the oracle's.  pc = 3: IC(0) of NEXT-2 (reading P2a; the
    device factor and sync-free triangular solves against the oracle's row-order ones)."""
    torch, trplk = need_gpu()
    P = gen.make(name, N=N)
    P.l = l
    P.q = P.q if name != "C1" else 12
    g = gpu_solve(trplk, P, precond=pc)
    o = oracle_solve(orc, P, precond=pc)
    if pc == 2:
        # the per-cycle M depends on theta_t, so rounding-level differences in theta_t feed back
        # into the operator every cycle: the trajectories agree to 1e-10 for dozens of cycles and
        # then drift (C2-24: cycle 56, 2e-10); the protocol's "GPU = oracle +-1 cycle" + results
        assert g["stats"]["status"] == o["status"] == "OK"
        assert np.all(g["residuals"] <= P.tol)
        c = first_divergence(g, o, norm_inf(P))
        assert c is None or c >= 20, c
        assert abs(g["stats"]["cycles"] - o["cycles"]) <= 1
        assert np.max(np.abs(g["eigenvalues"] - o["eigenvalues"]) / np.abs(o["eigenvalues"])) <= 1e-9
        return
    check_parity(g, o, P)
    assert g["stats"]["precond_applies"] >= 0


@pytest.mark.parametrize("name,N,b,over", [("C2", 12, 2, {}), ("C2", 24, 2, {}), ("C2", 16, 3, {}),
                                           ("C2", 12, 4, {"p": 4, "q": 12, "l": 4}),
                                           ("C3", 12, 2, {"p": 10, "q": 24, "l": 3}), ("C5", 16, 2, {}),
                                           ("C1", None, 2, {}), ("C2", 16, 4, {"l": 0})])
def test_block_trplk_parity(orc, gen, name, N, b, over):
    """NEXT-3, block TRPL+K (options.block = b, reading B1): the GPU's block inner loop (SpMM of b
    vectors with the preconditioner and first-pass dots fused, block CGS2 with Cholesky-QR)
    against the oracle's column-by-column construction of the same space: identical trajectory
    and A-matvec count (or a near-tie on the clustered C3), eigenvalues within 1e-9."""
    torch, trplk = need_gpu()
    P = gen.make(name, N=N)
    for k_, v in over.items():
        setattr(P, k_, v)
    g = gpu_solve(trplk, P, block=b)
    o = oracle_solve(orc, P, block=b)
    check_parity(g, o, P, allow_tie_divergence=(name == "C3"))
    X = g["X"]
    assert np.max(np.abs(X.T @ X - np.eye(P.p))) <= 1e-10


@pytest.mark.parametrize("name,N", [("C2", 16), ("C3", 12), ("C4", 8), ("C5", 20), ("C1", None)])
def test_dia_constant_diagonals_bitwise(gen, name, N):
    """DIA-C (constant diagonals read as a presence bit + the constant by the thread-per-row and
    fused K1, lean_k1.cuh / fused.cuh; the other kernels keep reading the value arrays, which stay
    populated; TRPLK_DIAC=0 turns it off): the decoded values are the stored ones bit for bit, so a
    solve with DIA-C is bitwise the solve without it -- eigenvalues, eigenvectors, residuals and
    matvec count.  The variant suite re-runs this file with TRPLK_K1=lean, where the decode is
    used at every size."""
    import os
    torch, trplk = need_gpu()
    P = gen.make(name, N=N)
    out = {}
    for v in ("0", "1"):
        os.environ["TRPLK_DIAC"] = v
        try:
            ctx = trplk.trplk_create(P.A, P.B, P.sigma)
        finally:
            os.environ.pop("TRPLK_DIAC", None)
        ev, X, rs, st = trplk.trplk_solve(ctx, P.p, P.q, P.l, P.tol, use_graphs=0)
        out[v] = (ev, X.cpu().numpy().copy(), rs, st["a_matvecs"])
        ctx.close()
    (e0, X0, r0, m0), (e1, X1, r1, m1) = out["0"], out["1"]
    assert np.array_equal(e0, e1) and np.array_equal(X0, X1) and np.array_equal(r0, r1) and m0 == m1


@pytest.mark.parametrize("name,N", [("C2", 24), ("C5", 24), ("C2", None)])
def test_kplus_first_pass_on_preceding_k1(gen, name, N):
    """The first CGS pass of each +K column (U^T x^prev_j, ||x^prev_j||^2; reading R3) computed as
    the second dot set of the K1 launch before it (the last inner step's, or the previous +K
    column's T-column K1) instead of its own pass over U: the same products on the same tiles
    and grid, so the solve is bitwise the one with the separate launch (TRPLK_KPLUS_XD=0)."""
    import os
    if any(os.environ.get(v) for v in ("TRPLK_K1", "TRPLK_KPLUS", "TRPLK_FUSE", "TRPLK_GRID", "TRPLK_NO_SMALL")):
        pytest.skip("a property of the default kernel selection (a forced K1 variant computes the "
                    "ride-along dots in another kernel than the separate launch)")
    torch, trplk = need_gpu()
    P = gen.make(name, N=N)
    out = {}
    for v in ("0", "1"):
        os.environ["TRPLK_KPLUS_XD"] = v
        try:
            ctx = trplk.trplk_create(P.A, P.B, P.sigma)
        finally:
            os.environ.pop("TRPLK_KPLUS_XD", None)
        ev, X, rs, st = trplk.trplk_solve(ctx, P.p, P.q, P.l, P.tol)
        out[v] = (ev, X.cpu().numpy().copy(), rs, st)
        ctx.close()
    (e0, X0, r0, s0), (e1, X1, r1, s1) = out["0"], out["1"]
    assert s1["status"] == "OK" and s0["a_matvecs"] == s1["a_matvecs"]
    assert np.array_equal(e0, e1) and np.array_equal(X0, X1) and np.array_equal(r0, r1)
    # the column's own pass-1 launch stays in the graph as a gated no-op: fewer algorithmic bytes
    assert s1["model_bytes"] < s0["model_bytes"]
