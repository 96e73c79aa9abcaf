"""The solver's kernels at a config's full size, launched alone through the kernel-level C ABI
(include/trplk_kernels.h), for ncu --set full captures (a full solve has thousands of launches,
too many for the profiler's interception) and standalone timing.
    python tools/kernels_at.py CONFIG k [reps]
  K1  trplk_k_step1 at width k      (inner-step K1: k_step1_pipe / k_step1_rs2)
  K2+K3 trplk_k_cgs2 at width k     (k_step1_rs2 first-pass dots with A absent, k_upd2_wp2, k_upd FINAL)
  K5  trplk_k_rotate k -> p columns (k_rotate_s)
  +K  trplk_k_block GRAM / UPD / SPMM with c = k_plus vectors (k_blk)"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402


def main(cfg, k, reps):
    from paper_1711_10128_b200 import build
    build.build()
    from paper_1711_10128_b200 import inputs, trplk
    P = inputs.make(cfg)
    n = P.A.n
    ctx = trplk.trplk_create(P.A, P.B, P.sigma)
    ld = ctx.ld
    kk = max(k, P.q)
    g = torch.Generator(device="cuda").manual_seed(5)
    U = torch.randn((kk, ld), dtype=torch.float64, device="cuda", generator=g) / np.sqrt(n)
    w = torch.zeros(ld, dtype=torch.float64, device="cuda")
    out = torch.zeros(ld, dtype=torch.float64, device="cuda")
    X = torch.zeros((P.p, ld), dtype=torch.float64, device="cuda")
    Y = np.random.default_rng(1).standard_normal((kk, P.p))
    c = max(P.l, 1)
    Yb = torch.randn((c, ld), dtype=torch.float64, device="cuda", generator=g)
    Yo = torch.zeros((c, ld), dtype=torch.float64, device="cuda")
    H = np.random.default_rng(2).standard_normal((k, c))
    torch.cuda.synchronize()
    for _ in range(reps):
        t0 = time.perf_counter()
        trplk.trplk_k_step1(ctx, U, ld, k, U[k - 1], 2.5, w)
        trplk.trplk_k_cgs2(ctx, U, ld, k, w, out)
        trplk.trplk_k_rotate(ctx, U, ld, kk, Y, P.p, X, ld)
        if P.B is None:
            trplk.trplk_k_block(ctx, 0, U, ld, k, Yb, ld, c)
            trplk.trplk_k_block(ctx, 1, U, ld, k, Yb, ld, c, Rinv=np.eye(c), H=H, Yout=Yo, ldyo=ld)
            trplk.trplk_k_block(ctx, 2, U, ld, k, Yb, ld, c)
        torch.cuda.synchronize()
        print(f"round {time.perf_counter() - t0:.4f} s", flush=True)
    ctx.close()


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]), int(sys.argv[3]) if len(sys.argv) > 3 else 2)
