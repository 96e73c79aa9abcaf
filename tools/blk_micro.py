"""Bandwidth of the block kernels (block.cuh) at the C5 size through trplk_k_block: GRAM / UPD /
SPMM of c vectors against k basis columns (tools/, measurement).
    python tools/blk_micro.py [k] [c] [reps]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402


def main(k, c, reps):
    from paper_1711_10128_b200 import build
    build.build()
    from paper_1711_10128_b200 import inputs, trplk
    P = inputs.make("C5")
    n = P.A.n
    ctx = trplk.trplk_create(P.A, None, 0.0)
    ld = ctx.ld
    g = torch.Generator(device="cuda").manual_seed(3)
    U = torch.randn((k, ld), dtype=torch.float64, device="cuda", generator=g)
    Y = torch.randn((c, ld), dtype=torch.float64, device="cuda", generator=g)
    Yo = torch.zeros((c, ld), dtype=torch.float64, device="cuda")
    H = np.random.default_rng(1).standard_normal((k, c))
    R = np.eye(c)
    for mode, name, byts in ((0, "GRAM", 8.0 * n * (k + c)), (1, "UPD", 8.0 * n * (k + 2 * c)),
                             (2, "SPMM", 8.0 * n * (k + c) + 56.0 * n)):
        kw = dict(Rinv=R, H=H, Yout=Yo, ldyo=ld) if mode == 1 else {}
        trplk.trplk_k_block(ctx, mode, U, ld, k, Y, ld, c, **kw)
        ts = []
        for _ in range(reps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            trplk.trplk_k_block(ctx, mode, U, ld, k, Y, ld, c, **kw)
            ts.append(time.perf_counter() - t0)
        t = min(ts)
        print(f"{name} k={k} c={c}: {t * 1e3:.3f} ms  {byts / t / 1e9:.0f} GB/s (incl. host sync)", flush=True)
    ctx.close()


if __name__ == "__main__":
    a = [int(x) for x in sys.argv[1:]]
    main(a[0] if a else 24, a[1] if len(a) > 1 else 2, a[2] if len(a) > 2 else 3)
