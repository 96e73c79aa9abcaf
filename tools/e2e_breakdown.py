"""Where the e2e time of bench.py goes (tools/): create / solve / D2H / destroy, host-timed."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1711_10128_b200 import build, inputs, trplk  # noqa: E402

build.build()
cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
P = inputs.make(cfg)
pin = [torch.from_numpy(a).pin_memory() for a in (P.A.rowptr, P.A.col, P.A.val)]


class H:
    def __init__(s, rp, c, v):
        s.rowptr, s.col, s.val, s.n, s.row_begin = rp.numpy(), c.numpy(), v.numpy(), P.A.n, 0


HA = H(*pin)
out = torch.empty((P.p, P.A.n), dtype=torch.float64).pin_memory()
for it in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ctx = trplk.trplk_create(HA, None, P.sigma)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    ev, _, rs, st = trplk.trplk_solve(ctx, P.p, P.q, P.l, P.tol, evecs_out=out)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    ctx.close()
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    print(f"{cfg} it{it}: create {1e3*(t1-t0):.1f} ms  solve+D2H {1e3*(t2-t1):.1f} ms  destroy {1e3*(t3-t2):.1f} ms",
          flush=True)
