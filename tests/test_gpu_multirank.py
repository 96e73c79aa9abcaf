"""Multi-rank z-slab solves on the GPU through the in-process loopback hub.

The row (z-slab) partition, ghost planning, halo exchange of g_j before every SpMV, and the
rank-ordered reduction of every dot/norm run exactly as with NCCL, except that the exchanges
are device-to-device copies ordered by CUDA events between the rank threads' streams (no
kernel waits on another rank, so several ranks can share the one GPU this run has).  Checked
against the 1-rank solve and the oracle (8(c.4) "Multi-GPU": same matvec count, eigenvalues
within 1e-10 relative) and for B-orthonormality of the gathered eigenvectors."""
import threading

import numpy as np
import pytest
import scipy.linalg as sla

from gpu_util import need_gpu

pytestmark = pytest.mark.gpu


def _rank_solve(trplk, inputs, name, N, hub, rank, nranks, out, **over):
    import torch
    torch.cuda.set_device(0)
    P0 = inputs.make(name, N=N, **over)
    n = P0.A.n
    plane = 1 if P0.grid["dim"] == 1 else N * N
    rb, re = inputs.slab_rows(n, nranks, rank, plane)
    P = inputs.make(name, N=N, row_begin=rb, row_end=re, **over)
    try:
        ctx = trplk.trplk_create(P.A, P.B, P.sigma, n_global=n, row_begin=rb, row_end=re,
                                 loopback=(hub, rank, nranks))
        ev, X, rs, st = trplk.trplk_solve(ctx, P.p, P.q, P.l, P.tol)
        log = trplk.trplk_get_log(ctx, ph=P.p)
        out[rank] = {"ev": ev, "X": X.cpu().numpy().copy(), "rs": rs, "st": st, "rows": (rb, re), "log": log}
        ctx.close()
    except Exception as e:  # reported by the main thread
        out[rank] = e


def _multirank(trplk, inputs, name, N, nranks, **over):
    hub = trplk.trplk_loopback_create(nranks)
    out = [None] * nranks
    th = [threading.Thread(target=_rank_solve, args=(trplk, inputs, name, N, hub, r, nranks, out), kwargs=over)
          for r in range(nranks)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    assert not any(t.is_alive() for t in th), "loopback ranks did not finish"
    trplk.trplk_loopback_destroy(hub)
    for o in out:
        if isinstance(o, Exception):
            raise o
    return out


@pytest.mark.parametrize("name,N,nranks", [("C2", 16, 2), ("C2", 16, 4), ("C4", 12, 2), ("C1", 200, 2)])
def test_loopback_ranks_match_one_rank(gen, orc, name, N, nranks):
    torch, trplk = need_gpu()
    P = gen.make(name, N=N)
    ctx = trplk.trplk_create(P.A, P.B, P.sigma)
    ev1, X1, rs1, st1 = trplk.trplk_solve(ctx, P.p, P.q, P.l, P.tol)
    log1 = trplk.trplk_get_log(ctx, ph=P.p)
    ctx.close()
    outs = _multirank(trplk, gen, name, N, nranks)
    # every rank reports the same (replicated) eigenvalues, counters and trajectory
    for o in outs[1:]:
        assert np.array_equal(o["ev"], outs[0]["ev"])
        assert o["st"]["a_matvecs"] == outs[0]["st"]["a_matvecs"]
        assert np.array_equal(o["log"]["theta_t"], outs[0]["log"]["theta_t"])
    o0 = outs[0]
    assert o0["st"]["status"] == "OK"
    # P ranks vs 1 rank: only the reduction order differs
    assert o0["st"]["a_matvecs"] == st1["a_matvecs"], (o0["st"]["a_matvecs"], st1["a_matvecs"])
    assert np.max(np.abs(o0["ev"] - ev1) / np.abs(ev1)) <= 1e-10
    # gathered eigenvectors: B-orthonormal, residuals recomputed on the host <= tol
    X = np.concatenate([o["X"] for o in outs], axis=0)
    A = P.A.to_scipy()
    B = None if P.B is None else P.B.to_scipy()
    BX = X if B is None else B @ X
    assert np.max(np.abs(X.T @ BX - np.eye(P.p))) <= 1e-10
    R = A @ X - BX * o0["ev"]
    assert np.all(np.linalg.norm(R, axis=0) <= P.tol * (1 + 1e-6))
    # and against the oracle (eigenvalues; the trajectory protocol is the 1-rank tests')
    ro = orc.solve(P.A, P.B, P.p, P.q, P.l, P.tol, P.sigma, want_vectors=False)
    assert np.max(np.abs(o0["ev"] - ro["eigenvalues"]) / np.abs(ro["eigenvalues"])) <= 1e-9
    # span agreement with the 1-rank eigenvectors per eigenvalue cluster
    X1h = X1.cpu().numpy()
    ev = o0["ev"]
    groups, g = [], [0]
    for i in range(1, P.p):
        if ev[i] - ev[i - 1] <= 1e-6 * abs(ev[i]):
            g.append(i)
        else:
            groups.append(g)
            g = [i]
    groups.append(g)
    for g in groups:
        M = X[:, g].T @ (X1h[:, g] if B is None else B @ X1h[:, g])
        s = np.linalg.svd(M, compute_uv=False)
        assert np.min(s) >= 1 - 1e-8, (g, s)


def _pl1_rank(trplk, inputs, name, N, hub, rank, nranks, out, m):
    import torch
    torch.cuda.set_device(0)
    P0 = inputs.make(name, N=N)
    n = P0.A.n
    plane = 1 if P0.grid["dim"] == 1 else N * N
    rb, re = inputs.slab_rows(n, nranks, rank, plane)
    P = inputs.make(name, N=N, row_begin=rb, row_end=re)
    try:
        ctx = trplk.trplk_create(P.A, P.B, P.sigma, n_global=n, row_begin=rb, row_end=re,
                                 loopback=(hub, rank, nranks))
        trplk.trplk_pl1_set_qopt(ctx, 40)  # the P7 diagnostic rides along (rank reductions)
        rho, res, x, st, log = trplk.trplk_pl1_solve(ctx, m, P.tol)
        out[rank] = {"rho": rho, "res": res, "x": x.cpu().numpy().copy(), "st": st, "log": log,
                     "qopt": trplk.trplk_pl1_get_qopt(ctx)}
        ctx.close()
    except Exception as e:  # reported by the main thread
        out[rank] = e


@pytest.mark.parametrize("name,N,nranks", [("C2", 16, 2), ("C4", 10, 2), ("C2", 16, 4)])
def test_pl1_loopback_ranks(gen, orc, name, N, nranks):
    """PL+1 on z-slab ranks (loopback hub): every rank reports the same rho / iterations; the
    same iteration and A-matvec counts as the oracle; gathered x = the oracle's x."""
    torch, trplk = need_gpu()
    m = 4
    hub = trplk.trplk_loopback_create(nranks)
    out = [None] * nranks
    th = [threading.Thread(target=_pl1_rank, args=(trplk, gen, name, N, hub, r, nranks, out, m))
          for r in range(nranks)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    assert not any(t.is_alive() for t in th)
    trplk.trplk_loopback_destroy(hub)
    for o in out:
        if isinstance(o, Exception):
            raise o
    for o in out[1:]:
        assert o["rho"] == out[0]["rho"] and o["st"]["cycles"] == out[0]["st"]["cycles"]
    P = gen.make(name, N=N)
    r = orc.pl1_solve(P.A, P.B, m=m, tol=P.tol, sigma=P.sigma, qopt_cap=40)
    o0 = out[0]
    for o in out[1:]:
        assert np.array_equal(o["qopt"]["rho_star"], o0["qopt"]["rho_star"])
    assert np.array_equal(o0["qopt"]["dim"], r["log"]["qdim"])
    rq = r["log"]["qopt"]
    assert np.max(np.abs(o0["qopt"]["rho_star"] - rq) / np.abs(rq)) <= 1e-10
    assert o0["st"]["status"] == "OK" and r["status"] == "OK"
    assert o0["st"]["cycles"] == r["cycles"] and o0["st"]["a_matvecs"] == r["a_matvecs"]
    assert abs(o0["rho"] - r["rho"]) <= 1e-12 * abs(r["rho"])
    x = np.concatenate([o["x"] for o in out])
    B = None if P.B is None else P.B.to_scipy()
    Bx = x if B is None else B @ x
    assert abs(abs(Bx @ r["x"]) - 1) <= 1e-8


@pytest.mark.parametrize("nranks", [2, 3])
def test_loopback_ranks_block_kplus(gen, nranks):
    """k_plus = 3: the +K block path (block.cuh: GRAM / UPD / SPMM reductions through the rank
    allgather + rank-ordered finalize, halo of the appended block) on 2 and 3 ranks reproduces the
    1-rank solve (same trajectory and A-matvec count, eigenvalues within 1e-10)."""
    torch, trplk = need_gpu()
    P = gen.make("C2", N=15, l=3)
    ctx = trplk.trplk_create(P.A, P.B, P.sigma)
    ev1, X1, rs1, st1 = trplk.trplk_solve(ctx, P.p, P.q, P.l, P.tol)
    log1 = trplk.trplk_get_log(ctx, ph=P.p)
    ctx.close()
    outs = _multirank(trplk, gen, "C2", 15, nranks, l=3)
    o0 = outs[0]
    assert o0["st"]["status"] == "OK"
    assert o0["st"]["a_matvecs"] == st1["a_matvecs"]
    assert list(o0["log"]["nprev"]) == list(log1["nprev"]) and max(log1["nprev"]) == 3
    assert np.max(np.abs(o0["ev"] - ev1) / np.abs(ev1)) <= 1e-10


@pytest.mark.parametrize("name,N,nranks", [("C2", 24, 2), ("C5", 24, 3)])
def test_loopback_halo_overlap(gen, orc, name, N, nranks):
    """Halo overlap (engine run_k1_overlap): the exchange of g's boundary rows on a side stream
    while K1 covers the interior rows, then K1 over the two boundary row ranges -- three launches
    feeding one grid reduction.  Against the exchange-first K1 (TRPLK_HALO_OVERLAP=0): same matvec
    count and trajectory structure, eigenvalues within 1e-10 relative (only the reduction's CTA
    grouping differs), and against the oracle within 1e-9."""
    import os
    torch, trplk = need_gpu()
    os.environ["TRPLK_HALO_OVERLAP"] = "0"
    try:
        off = _multirank(trplk, gen, name, N, nranks)
    finally:
        os.environ.pop("TRPLK_HALO_OVERLAP", None)
    on = _multirank(trplk, gen, name, N, nranks)
    a, b = on[0], off[0]
    assert a["st"]["status"] == b["st"]["status"] == "OK"
    assert a["st"]["a_matvecs"] == b["st"]["a_matvecs"]
    for key in ("t", "k", "nprev"):
        assert np.array_equal(a["log"][key], b["log"][key]), key
    assert np.max(np.abs(a["ev"] - b["ev"]) / np.abs(b["ev"])) <= 1e-10
    for o in on[1:]:
        assert np.array_equal(o["ev"], a["ev"])
    P = gen.make(name, N=N)
    ro = orc.solve(P.A, P.B, P.p, P.q, P.l, P.tol, P.sigma, want_vectors=False)
    assert np.max(np.abs(a["ev"] - ro["eigenvalues"]) / np.abs(ro["eigenvalues"])) <= 1e-9
    assert np.all(a["rs"] <= P.tol)
