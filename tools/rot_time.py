"""Time the K5 rotation X = U Y alone at a config's size through the kernel ABI (trplk_k_rotate),
CUDA events, 512 MB flush between launches, median of reps (tools/, not product).

    python tools/rot_time.py C3 48 20 [reps]      # config, k, ncol"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1711_10128_b200 import build, inputs, trplk  # noqa: E402

build.build()
cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
k = int(sys.argv[2]) if len(sys.argv) > 2 else 48
ncol = int(sys.argv[3]) if len(sys.argv) > 3 else 20
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 20
P = inputs.make(cfg)
n = P.A.n
ctx = trplk.trplk_create(P.A, P.B, P.sigma)
ld = ctx.ld
g = torch.Generator(device="cuda").manual_seed(5)
U = torch.randn((k, ld), dtype=torch.float64, device="cuda", generator=g)
Y = np.random.default_rng(1).standard_normal((k, ncol))
X = torch.zeros((ncol, ld), dtype=torch.float64, device="cuda")
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float64, device="cuda")
ts = []
for r in range(reps + 2):
    flush.fill_(1.0)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    trplk.trplk_k_rotate(ctx, U, ld, k, Y, ncol, X, ld)
    e1.record()
    torch.cuda.synchronize()
    if r >= 2:
        ts.append(e0.elapsed_time(e1))
ms = float(np.median(ts))
by = 8.0 * n * (k + ncol)
print(f"{cfg} rotation k={k} ncol={ncol}: {ms * 1e3:.1f} us median (min {min(ts) * 1e3:.1f}), "
      f"{by / 1e9:.3f} GB -> {by / ms / 1e6:.0f} GB/s")
ctx.close()
