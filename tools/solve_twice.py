"""Two solves of one config; the second inside the NVTX range "timed" (for ncu --nvtx-include
timed/ launch lists of exactly one solve).  tools/, not product."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1711_10128_b200 import build, inputs, trplk  # noqa: E402

build.build()
P = inputs.make(sys.argv[1] if len(sys.argv) > 1 else "C2")
ctx = trplk.trplk_create(P.A, P.B, P.sigma)
for i in range(2):
    if i == 1:
        torch.cuda.nvtx.range_push("timed")
    ev, X, rs, st = trplk.trplk_solve(ctx, P.p, P.q, P.l, P.tol)
    torch.cuda.synchronize()
    if i == 1:
        torch.cuda.nvtx.range_pop()
    print(i, st["a_matvecs"], st["kernel_launches"], f"{st['solve_seconds'] * 1e3:.2f} ms", flush=True)
ctx.close()
