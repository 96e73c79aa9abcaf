"""Time the inner-step K1 alone at a config's size through the kernel ABI (trplk_k_step1), the
variant chosen by TRPLK_K1 / TRPLK_DIAC in the environment (tools/, not product).

    TRPLK_K1=lean python tools/k1_time.py C5 15 [reps]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1711_10128_b200 import build, inputs, trplk  # noqa: E402

build.build()
cfg = sys.argv[1] if len(sys.argv) > 1 else "C5"
k = int(sys.argv[2]) if len(sys.argv) > 2 else 15
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 20
P = inputs.make(cfg)
n = P.A.n
ctx = trplk.trplk_create(P.A, P.B, P.sigma)
info = trplk.trplk_info(ctx)
ld = ctx.ld
g = torch.Generator(device="cuda").manual_seed(5)
U = torch.randn((k + 1, ld), dtype=torch.float64, device="cuda", generator=g) / np.sqrt(n)
w = torch.zeros(ld, dtype=torch.float64, device="cuda")
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float64, device="cuda")
ts = []
for r in range(reps + 2):
    flush.fill_(1.0)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    out = trplk.trplk_k_step1(ctx, U, ld, k, U[k - 1], 2.5, w)
    e1.record()
    torch.cuda.synchronize()
    if r >= 2:
        ts.append(e0.elapsed_time(e1))
ms = float(np.median(ts))
by = info["sell_bytes_a"] + 8.0 * n * (k + 2)
print(f"{cfg} k={k} K1[{os.environ.get('TRPLK_K1', 'default')}, DIAC={os.environ.get('TRPLK_DIAC', '0')}]: "
      f"{ms:.3f} ms median (min {min(ts):.3f}), {by / 1e9:.2f} GB -> {by / ms / 1e6:.0f} GB/s")
ctx.close()
