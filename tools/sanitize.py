"""Small solves for compute-sanitizer (tools/): C1 (n=200), C2 (12^3), C4 (8^3 pencil), all through
trplk_solve, plus the loopback 2-rank path.   compute-sanitizer --tool memcheck python tools/sanitize.py"""
import os
import sys
import threading

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1711_10128_b200 import build, inputs, trplk  # noqa: E402

build.build()
torch.cuda.set_device(0)
for name, N in (("C1", 200), ("C2", 12), ("C4", 8), ("C3", 10)):
    P = inputs.make(name, N=N)
    ctx = trplk.trplk_create(P.A, P.B, P.sigma)
    for graphs in (1, 0):
        ev, X, rs, st = trplk.trplk_solve(ctx, P.p, P.q, P.l, P.tol, use_graphs=graphs)
        print(name, "graphs" if graphs else "eager", st["status"], st["a_matvecs"], float(np.max(rs)), flush=True)
    ctx.close()
# two loopback ranks
P0 = inputs.make("C2", N=12)
n = P0.A.n
hub = trplk.trplk_loopback_create(2)
res = [None, None]


def rank(r):
    torch.cuda.set_device(0)
    rb, re = inputs.slab_rows(n, 2, r, 144)
    P = inputs.make("C2", N=12, row_begin=rb, row_end=re)
    ctx = trplk.trplk_create(P.A, P.B, P.sigma, n_global=n, row_begin=rb, row_end=re, loopback=(hub, r, 2))
    res[r] = trplk.trplk_solve(ctx, P.p, P.q, P.l, P.tol)[3]["a_matvecs"]
    ctx.close()


th = [threading.Thread(target=rank, args=(r,)) for r in range(2)]
[t.start() for t in th]
[t.join() for t in th]
trplk.trplk_loopback_destroy(hub)
print("loopback ranks", res, flush=True)
