"""The opt-in RR eigensolver TRPLK_EIG=tri (eig_tri.cu: tridiagonalisation + multisection +
inverse iteration) against LAPACK and inside a full solve against the oracle.  The switch is
read once per process, so each check runs in a child process."""
import os
import subprocess
import sys

import pytest

from gpu_util import need_gpu

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r'''
import sys, numpy as np
sys.path.insert(0, ROOT); sys.path.insert(0, ROOT + "/tests")
from paper_1711_10128_b200 import build, inputs, trplk
import oracle
build.build(); oracle.build()
P = inputs.make("C1")
ctx = trplk.trplk_create(P.A)
rng = np.random.default_rng(7)
cases = []
for k in (2, 3, 17, 30, 48, 64):
    M = rng.standard_normal((k, k)); cases.append(M + M.T)
# exact multiplicities and a graded spectrum
Q, _ = np.linalg.qr(rng.standard_normal((24, 24)))
cases.append(Q @ np.diag(np.repeat([1.0, 2.0, 2.5, 4.0], 6)) @ Q.T)
cases.append(Q @ np.diag(np.logspace(-8, 2, 24)) @ Q.T)
for T in cases:
    k = T.shape[0]
    th, Y = trplk.trplk_k_sym_eig(ctx, T)
    ref = np.linalg.eigvalsh(T)
    sc = np.max(np.abs(ref))
    assert np.max(np.abs(th - ref)) <= 1e-13 * sc, (k, np.max(np.abs(th - ref)))
    assert np.max(np.abs(Y.T @ Y - np.eye(k))) <= 1e-12, k
    assert np.max(np.abs(T @ Y - Y * th)) <= 1e-13 * sc, k
ctx.close()
for name, N, over in (("C2", 16, {}), ("C3", 12, {"p": 10, "q": 24, "l": 3}), ("C4", 8, {})):
    P = inputs.make(name, N=N, **over)
    ctx = trplk.trplk_create(P.A, P.B, P.sigma)
    ev, X, rs, st = trplk.trplk_solve(ctx, P.p, P.q, P.l, P.tol)
    ctx.close()
    o = oracle.solve(P.A, P.B, P.p, P.q, P.l, P.tol, P.sigma, want_vectors=False)
    assert st["status"] == "OK" and o["status"] == "OK"
    assert np.all(rs <= P.tol)
    assert np.max(np.abs(ev - o["eigenvalues"]) / np.abs(o["eigenvalues"])) <= 1e-9, name
print("tri OK")
'''


def test_eig_tri_child():
    need_gpu()
    env = dict(os.environ, TRPLK_EIG="tri")
    r = subprocess.run([sys.executable, "-c", CHILD.replace("ROOT", repr(ROOT))], env=env, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0 and "tri OK" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]
