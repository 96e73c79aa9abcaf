"""Worker of tests/test_gpu_torchrun.py (launched by torch.distributed.run, one process per rank,
all on the box's one GPU): per-rank z-slab generation, trplk_create with host-staged exchanges
over the gloo process group (comm='host'), a full solve; rank 0 writes the result as JSON."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402


def main(cfg, N, out):
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    torch.cuda.set_device(0)
    from paper_1711_10128_b200 import build
    build.build()
    from paper_1711_10128_b200 import inputs, trplk
    full = inputs.make(cfg, N=N)
    n = full.A.n
    plane = 1 if full.grid["dim"] == 1 else N * N
    rb, re = inputs.slab_rows(n, world, rank, plane)
    P = inputs.make(cfg, N=N, row_begin=rb, row_end=re)
    ctx = trplk.trplk_create(P.A, P.B, P.sigma, n_global=n, row_begin=rb, row_end=re, group=dist.group.WORLD,
                             comm="host")
    ev, X, rs, st = trplk.trplk_solve(ctx, P.p, P.q, P.l, P.tol)
    log = trplk.trplk_get_log(ctx, ph=P.p)
    xs = [None] * world
    dist.all_gather_object(xs, X.cpu().numpy())
    if rank == 0:
        json.dump({"eigenvalues": ev.tolist(), "residuals": rs.tolist(), "stats": {k: (v if not isinstance(v, float) else float(v)) for k, v in st.items()},
                   "t": list(map(int, log["t"])), "k": list(map(int, log["k"])), "theta_t": list(map(float, log["theta_t"])),
                   "nranks": world, "X": np.concatenate(xs, axis=0).tolist()}, open(out, "w"))
    ctx.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]), sys.argv[3])
