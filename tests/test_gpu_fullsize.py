"""Full-size parity with the oracle at BASELINE.json sizes, in the launch configuration bench.py
times.  The oracle's full solves for C2-C4 take minutes to hours on a CPU, so their results are
committed as tests/golden/oracle_<cfg>.json (written by tests/golden/make_oracle_golden.py,
which calls only oracle/).  C5 (n = 1.3e8) is checked through properties that hold at any size:
residuals recomputed independently on the host, B-orthonormality, Weyl bounds and the oracle's
SpMV on sampled rows."""
import json
import os

import numpy as np
import pytest

from gpu_util import need_gpu

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _gold(name):
    p = os.path.join(GOLD, f"oracle_{name}.json")
    if not os.path.exists(p):
        pytest.skip(f"{p} not generated yet")
    return json.load(open(p))


def _solve(trplk, P):
    ctx = trplk.trplk_create(P.A, P.B, P.sigma)
    ev, X, rs, st = trplk.trplk_solve(ctx, P.p, P.q, P.l, P.tol)
    log = trplk.trplk_get_log(ctx, ph=P.p)
    return ctx, ev, X, rs, st, log


def _near_tie(thetas, res, tol):
    th = np.asarray(thetas)
    return bool(np.any(np.abs(np.diff(th)) <= 1e-10 * np.abs(th[1:])) or abs(res - tol) <= 1e-2 * tol)


def _emergence(log, c):
    """Cycle c of a run is an emergence event (reading R17): with the target t unchanged, theta_t
    fell by more than the previous residual ||r_t||, i.e. by more than the distance from the old
    Ritz value to the nearest eigenvalue, so the Ritz value moved to ANOTHER eigenvalue.  For an
    exactly degenerate spectrum (C3: multiplicities 3 and 6) the Krylov space grows a new copy of
    a cluster only from rounding-level components, so when that happens depends on the rounding
    of the run, not on the method; the trajectories may part there."""
    if c == 0 or log["t"][c] != log["t"][c - 1]:
        return False
    return log["theta_t"][c - 1] - log["theta_t"][c] > log["res"][c - 1]


@pytest.mark.parametrize("name", ["C2", "C3", "C4", "C5"])
def test_fullsize_vs_oracle_golden(gen, name):
    torch, trplk = need_gpu()
    g = _gold(name)
    if name == "C5" and torch.cuda.get_device_properties(0).total_memory < 120e9:
        pytest.skip("needs ~80 GB of device memory")
    P = gen.make(name)
    ctx, ev, X, rs, st, log = _solve(trplk, P)
    assert st["status"] == "OK" and g["status"] == "OK"
    assert np.all(rs <= P.tol)
    ref = np.array(g["eigenvalues"])
    assert np.max(np.abs(ev - ref) / np.abs(ref)) <= 1e-9
    # trajectory: identical (t, width, X^prev width) and theta_t until a near-tie divergence
    A = P.A.to_scipy()
    nA = float(abs(A).sum(axis=1).max())
    lo = g["log"]
    n = min(len(lo["t"]), len(log["t"]))
    for c in range(n):
        same = (lo["t"][c] == log["t"][c] and lo["k"][c] == log["k"][c] and lo["nprev"][c] == log["nprev"][c]
                and abs(lo["theta_t"][c] - log["theta_t"][c]) <= 1e-10 * abs(lo["theta_t"][c]) + 1e-13 * nA)
        if not same:
            ok = _near_tie(g["log_thetas"][c], lo["res"][c], P.tol) or any(
                _emergence(L, cc) for L in (lo, log) for cc in range(max(c - 1, 1), min(c + 2, n)))
            assert ok, f"diverged at cycle {c} without a near-tie or an emergence event"
            # reported, and bounded: after the divergence both runs converge to the same clusters;
            # the total work may differ by the cycles the later emergence costs (<= 5 %)
            print(f"{name}: trajectories part at cycle {c} (t {lo['t'][c]} / {log['t'][c]}, theta_t "
                  f"{lo['theta_t'][c]:.16e} / {log['theta_t'][c]:.16e}); cycles oracle {g['cycles']} GPU "
                  f"{st['cycles']}, A-matvecs {g['a_matvecs']} / {st['a_matvecs']}")
            assert abs(st["cycles"] - g["cycles"]) <= 0.05 * g["cycles"]
            break
    else:
        assert st["a_matvecs"] == g["a_matvecs"]
    # B-orthonormality of the returned block
    Xh = X.cpu().numpy()
    BX = Xh if P.B is None else P.B.to_scipy() @ Xh
    assert np.max(np.abs(Xh.T @ BX - np.eye(P.p))) <= 1e-10
    # eigenvector entries at the oracle's sampled rows (golden files that carry them): for a
    # simple eigenvalue x is unique up to sign, and |x_gpu(i) - x_orc(i)| <= ||x_gpu - x_orc||_2
    # <= the angle, so north_star's angle bound 1e-6 caps every sampled entry
    if "sample_rows" in g and name != "C3":
        rows = np.array(g["sample_rows"])
        S = np.array(g["sample_vectors"]).T  # [n_sample, p]
        ev_o = np.array(g["eigenvalues"])
        for i in range(P.p):
            simple = all(abs(ev_o[i] - ev_o[j]) > 1e-9 * abs(ev_o[i]) for j in range(P.p) if j != i)
            if not simple:
                continue
            xs = Xh[rows, i]
            sg = 1.0 if np.dot(xs, S[:, i]) >= 0 else -1.0
            assert np.max(np.abs(sg * xs - S[:, i])) <= 1e-6, (name, i)
    ctx.close()


def test_C3_closed_form_clusters(gen):
    """128^3 Laplacian: the 20 smallest eigenvalues are complete clusters of the closed form."""
    torch, trplk = need_gpu()
    P = gen.make("C3")
    ctx, ev, X, rs, st, log = _solve(trplk, P)
    c = 2 - 2 * np.cos(np.arange(1, 129) * np.pi / 129)
    ref = np.sort(np.add.outer(np.add.outer(c[:8], c[:8]), c[:8]).ravel())[:20]
    assert st["status"] == "OK"
    # a-posteriori: |theta - lambda| <= ||r||^2 / gap with inter-cluster gap >= 5.8e-4, plus the
    # rounding floor of a backward-stable Rayleigh-Ritz, O(eps ||A||): 1e-14 ||A||_2 (||A||_2 < 12)
    assert np.all(np.abs(ev - ref) <= rs ** 2 / 5.8e-4 + 1e-14 * 12.0)
    ctx.close()


def test_C5_properties_at_full_size(orc, gen):
    """512^3 (n = 1.3e8) on one GPU: residuals recomputed on the host with the oracle's SpMV,
    B-orthonormality, Weyl bounds lambda_k(L) <= theta_k <= lambda_k(L) + 10."""
    torch, trplk = need_gpu()
    if torch.cuda.get_device_properties(0).total_memory < 120e9:
        pytest.skip("needs ~80 GB of device memory")
    P = gen.make("C5")
    ctx, ev, X, rs, st, log = _solve(trplk, P)
    assert st["status"] == "OK", st
    assert np.all(rs <= P.tol)
    Xh = X.cpu().numpy()
    G = Xh.T @ Xh
    assert np.max(np.abs(G - np.eye(P.p))) <= 1e-10
    for i in range(P.p):
        r = orc.spmv(P.A, Xh[:, i]) - ev[i] * Xh[:, i]
        assert abs(np.linalg.norm(r) - rs[i]) <= 1e-3 * P.tol + 1e-12
    c = 2 - 2 * np.cos(np.arange(1, 9) * np.pi / 513)
    lamL = np.sort(np.add.outer(np.add.outer(c, c), c).ravel())[:P.p]
    assert np.all(lamL <= ev + 1e-12) and np.all(ev <= lamL + 10.0)
    ctx.close()


def test_C3_eigenvectors_vs_exact_and_oracle(gen):
    """Full-size eigenvector parity on the clustered C3 through the exact
    eigenspaces (tests/closed_form.py, the sine tensor basis): at tol_parity = 1e-11 the GPU's
    vectors of every complete cluster lie within sin-angle ||r|| / gap (gap >= 5.8e-4 between
    clusters) of the exact eigenspace, computed on the FULL vectors here; the oracle's full vectors
    were measured the same way when tests/golden/oracle_C3_tol1e-11.json was written.  By the
    triangle inequality the GPU-oracle angle per cluster is at most the sum: <= 1e-6 required."""
    import sys
    torch, trplk = need_gpu()
    g = _gold("C3_tol1e-11")
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from closed_form import laplace3d_lowest, sin_angle
    P = gen.make("C3")
    ctx = trplk.trplk_create(P.A, P.B, P.sigma)
    ev, X, rs, st = trplk.trplk_solve(ctx, P.p, P.q, P.l, 1e-11)
    assert st["status"] == "OK" and np.all(rs <= 1e-11)
    lam, V, groups = laplace3d_lowest(128, P.p)
    assert groups == g["exact_groups"]
    Xh = X.cpu().numpy()
    for gi, grp in enumerate(groups):
        s_gpu = sin_angle(Xh[:, grp], V[:, grp])
        assert s_gpu <= np.max(rs[grp]) * np.sqrt(len(grp)) / 5.8e-4 + 1e-12, (grp, s_gpu)
        assert s_gpu + g["exact_sin_angle"][gi] <= 1e-6, (grp, s_gpu, g["exact_sin_angle"][gi])
    assert np.max(np.abs(ev - lam) / lam) <= 1e-9
    ctx.close()


def test_C4_eigenvectors_tol_parity_sampled(gen):
    """C4 (generalized pencil, random d) at tol_parity = 1e-11: eigenvalues within 1e-9 of the
    oracle's tol-parity run, and the B-normalised eigenvectors at the oracle's sampled rows within
    1e-6 (sign fixed per vector; every C4 eigenvalue here is simple)."""
    torch, trplk = need_gpu()
    g = _gold("C4_tol1e-11")
    P = gen.make("C4")
    ctx = trplk.trplk_create(P.A, P.B, P.sigma)
    ev, X, rs, st = trplk.trplk_solve(ctx, P.p, P.q, P.l, 1e-11)
    assert st["status"] == "OK" and np.all(rs <= 1e-11)
    ref = np.array(g["eigenvalues"])
    assert np.max(np.abs(ev - ref) / ref) <= 1e-9
    rows = np.array(g["sample_rows"])
    S = np.array(g["sample_vectors"]).T
    Xh = X.cpu().numpy()
    worst = 0.0
    for i in range(P.p):
        xs = Xh[rows, i]
        sg = 1.0 if np.dot(xs, S[:, i]) >= 0 else -1.0
        worst = max(worst, float(np.max(np.abs(sg * xs - S[:, i]))))
    assert worst <= 1e-6, worst
    ctx.close()
