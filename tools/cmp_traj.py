"""Grid-path vs multi-kernel vs oracle trajectory comparison (tools/, test infrastructure)."""
import sys, numpy as np
sys.path.insert(0, "."); sys.path.insert(0, "./tests")
from paper_1711_10128_b200 import build, inputs, trplk
import oracle; oracle.build()
build.build()
N = int(sys.argv[1]) if len(sys.argv) > 1 else 24
q = int(sys.argv[2]) if len(sys.argv) > 2 else 22
P = inputs.make("C2", N=N, q=q)
o = oracle.solve(P.A, P.B, P.p, P.q, P.l, P.tol, P.sigma, want_vectors=False)
lo = o["log"]
for dbg in (0, 2):
    ctx = trplk.trplk_create(P.A, P.B, P.sigma)
    if dbg: trplk.trplk_set_debug(ctx, dbg)
    ev, X, rs, st = trplk.trplk_solve(ctx, P.p, P.q, P.l, P.tol)
    lg = trplk.trplk_get_log(ctx, ph=P.p)
    n = min(len(lg["t"]), len(lo["t"]))
    rel = [abs(lg["theta_t"][c] - lo["theta_t"][c]) / abs(lo["theta_t"][c]) for c in range(n)]
    first = next((c for c in range(n) if lg["t"][c] != lo["t"][c] or lg["k"][c] != lo["k"][c]), None)
    print("debug", dbg, "matvecs", st["a_matvecs"], o["a_matvecs"], "cycles", len(lg["t"]), len(lo["t"]),
          "first struct div", first, "max rel theta diff", max(rel), "at", int(np.argmax(rel)))
    if first is not None:
        for c in range(max(0, first - 2), min(n, first + 2)):
            th = lo["thetas"][c]
            gap = float(np.min(np.abs(np.diff(th)) / np.abs(th[1:])))
            print("  cycle", c, "gpu t,k,res", lg["t"][c], lg["k"][c], lg["res"][c], "oracle", lo["t"][c], lo["k"][c],
                  lo["res"][c], "tol", P.tol, "min rel Ritz gap", gap)
    ctx.close()
