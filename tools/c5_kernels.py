"""The inner-step kernels at the C5 size, launched alone through the kernel-level C ABI
(include/trplk_kernels.h) -- for ncu --set full captures (a full C5 solve has ~5,700 launches, too
many to run under the profiler's interception).  Same instantiations the C5 solve runs:
  K1  trplk_k_step1 at k = 15           -> k_step1_lean<16, 1, 0> (z = A g, w = M(z - rho g), U^T [z w]; DIA-C)
  K1  trplk_k_step1 at k = 23           -> k_step1_rs2<24, 1>
  K2  trplk_k_cgs2 at k = 15, pass 2    -> k_upd2_wp2<8, 2>     (w' = w - U h1, U^T w', ||w'||^2)
  K3  trplk_k_cgs2 at k = 15, final     -> k_upd<16, 0>         (g = (w' - U h2) / beta)
  +K  trplk_k_cgs2 at k = 23, pass 1    -> k_step1_tp<24, 1, 0, 0> (U^T x, the +K / seed dots)
  K5  trplk_k_rotate k = 24, 8 columns  -> k_rotate_s<1, 24>    (X = U Y on DMMA)
    python tools/c5_kernels.py [reps]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402


def main(reps):
    from paper_1711_10128_b200 import build
    build.build()
    from paper_1711_10128_b200 import inputs, trplk
    P = inputs.make("C5")
    n = P.A.n
    ctx = trplk.trplk_create(P.A, P.B, P.sigma)
    ld = ctx.ld
    g = torch.Generator(device="cuda").manual_seed(5)
    U = torch.randn((24, ld), dtype=torch.float64, device="cuda", generator=g) / np.sqrt(n)
    w = torch.zeros(ld, dtype=torch.float64, device="cuda")
    out = torch.zeros(ld, dtype=torch.float64, device="cuda")
    X = torch.zeros((8, ld), dtype=torch.float64, device="cuda")
    Y = np.random.default_rng(1).standard_normal((24, 8))
    torch.cuda.synchronize()
    for _ in range(reps):
        t0 = time.perf_counter()
        trplk.trplk_k_step1(ctx, U, ld, 15, U[14], 2.5, w)
        trplk.trplk_k_cgs2(ctx, U, ld, 15, w, out)
        trplk.trplk_k_cgs2(ctx, U, ld, 23, w, out)
        trplk.trplk_k_rotate(ctx, U, ld, 24, Y, 8, X, ld)
        trplk.trplk_k_step1(ctx, U, ld, 23, U[22], 2.5, w)  # k > 16: k_step1_rs2<24, 1>
        torch.cuda.synchronize()
        print(f"round {time.perf_counter() - t0:.3f} s", flush=True)
    ctx.close()


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 2)
