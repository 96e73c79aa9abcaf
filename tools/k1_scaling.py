"""K1/K2/K3 live-profile time per launch vs problem size (C2 shape): fixed cost + bytes/BW.
tools/, not product."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1711_10128_b200 import build, inputs, trplk  # noqa: E402

build.build()
for N in (8, 16, 24, 32, 48, 64, 96):
    P = inputs.make("C2", N=N)
    ctx = trplk.trplk_create(P.A, P.B, P.sigma)
    trplk.trplk_solve(ctx, P.p, P.q, P.l, P.tol)
    trplk.trplk_profile(ctx, True)
    trplk.trplk_solve(ctx, P.p, P.q, P.l, P.tol)
    trplk.trplk_solve(ctx, P.p, P.q, P.l, P.tol)
    pr = trplk.trplk_profile_read(ctx)
    trplk.trplk_profile(ctx, False)
    ev, X, rs, st = trplk.trplk_solve(ctx, P.p, P.q, P.l, P.tol)
    c = max(pr["count"], 1)
    ms = pr["ms"] / c
    by = pr["bytes"] / c
    print(f"N={N:3d} n={P.A.n:8d} solve {st['solve_seconds']*1e3:8.2f} ms  K1 {ms[0]*1e3:6.2f} us ({by[0]/ms[0]/1e6:7.1f} GB/s)"
          f"  K2 {ms[1]*1e3:6.2f} us  K3 {ms[2]*1e3:6.2f} us  MB/launch K1 {by[0]/1e6:7.2f}", flush=True)
    ctx.close()
