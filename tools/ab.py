"""Interleaved A/B timing of two library configurations on one config (tools/, not product).

    python tools/ab.py C3 "TRPLK_DIAC=0" "" [rounds]

Each side's environment is set while its context is created (the switches read at create time:
TRPLK_DIAC, TRPLK_FUSE); solves alternate A B A B ... so clock / power drift hits both sides."""
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1711_10128_b200 import build, inputs, trplk  # noqa: E402


def env_of(spec):
    return dict(kv.split("=", 1) for kv in spec.split(",") if kv)


def create(P, spec):
    env = env_of(spec)
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        return trplk.trplk_create(P.A, P.B, P.sigma)
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


build.build()
cfg, sa, sb = sys.argv[1], sys.argv[2], sys.argv[3]
rounds = int(sys.argv[4]) if len(sys.argv) > 4 else 3
P = inputs.make(cfg)
ctx = {"A": create(P, sa), "B": create(P, sb)}
times = {"A": [], "B": []}
res = {}
for r in range(rounds + 1):
    for side in ("A", "B"):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ev, X, rs, st = trplk.trplk_solve(ctx[side], P.p, P.q, P.l, P.tol)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        if r > 0:
            times[side].append(dt * 1e3)
        res[side] = (ev, st["a_matvecs"], st["cycles"], st["kernel_launches"])
        del X
for side, spec in (("A", sa), ("B", sb)):
    t = times[side]
    print(f"{cfg} {side} [{spec or 'default'}]: median {statistics.median(t):.2f} ms  min {min(t):.2f}  all "
          f"{[round(x, 2) for x in t]}  matvecs {res[side][1]} cycles {res[side][2]} launches {res[side][3]}")
ea, eb = res["A"][0], res["B"][0]
print(f"{cfg} max rel eig diff A vs B: {np.max(np.abs(ea - eb) / np.abs(ea)):.3e}")
for c in ctx.values():
    c.close()
