"""The multi-process path on the one GPU of the box: torch.distributed.run starts 2
ranks, each generates its own z-slab, trplk_create bootstraps the partition through the process
group with host-staged exchanges (gloo, comm='host': no kernel waits on another rank, so two
processes can share one GPU), and the solve must reproduce the 1-rank solve (same trajectory and
A-matvec count, eigenvalues within 1e-10, B-orthonormal gathered eigenvectors with residuals <=
tol).  The NCCL transport itself needs >= 2 GPUs and is not run here.  bench.py's N = 2 path runs
the same way (--comm host)."""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

from gpu_util import need_gpu

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _torchrun(args, nproc=2, timeout=900):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr=127.0.0.1", f"--master-port={_port()}", *args]
    return subprocess.run(cmd, capture_output=True, text=True, timeout=timeout, cwd=ROOT)


@pytest.mark.parametrize("cfg,N", [("C2", 16), ("C4", 10)])
def test_two_processes_one_gpu_host_comm(gen, tmp_path, cfg, N):
    torch, trplk = need_gpu()
    out = str(tmp_path / "r.json")
    r = _torchrun([os.path.join(HERE, "_torchrun_solve.py"), cfg, str(N), out])
    assert r.returncode == 0, (r.stdout + r.stderr)[-3000:]
    g = json.load(open(out))
    P = gen.make(cfg, N=N)
    ctx = trplk.trplk_create(P.A, P.B, P.sigma)
    ev1, X1, rs1, st1 = trplk.trplk_solve(ctx, P.p, P.q, P.l, P.tol)
    log1 = trplk.trplk_get_log(ctx, ph=P.p)
    ctx.close()
    assert g["nranks"] == 2 and g["stats"]["status"] == "OK"
    assert g["t"] == list(log1["t"]) and g["k"] == list(log1["k"])
    assert g["stats"]["a_matvecs"] == st1["a_matvecs"]
    assert np.max(np.abs(np.array(g["eigenvalues"]) - ev1) / np.abs(ev1)) <= 1e-10
    X = np.array(g["X"])
    BX = X if P.B is None else P.B.to_scipy() @ X
    assert np.max(np.abs(X.T @ BX - np.eye(P.p))) <= 1e-10
    A = P.A.to_scipy()
    for i in range(P.p):
        ri = np.linalg.norm(A @ X[:, i] - g["eigenvalues"][i] * BX[:, i])
        assert ri <= P.tol * 1.01


def test_bench_two_ranks_host_comm():
    """bench.py --gpus 2 under torch.distributed.run (the driver's N > 1 launch), host-staged
    exchanges: rank 0 prints one JSON line with n_gpus = 2 and the 1-rank matvec count."""
    need_gpu()
    r = _torchrun(["bench.py", "--gpus", "2", "--comm", "host", "--config", "C2", "--steps", "1", "--warmup", "1",
                   "--no-e2e", "--no-cpu-baseline"])
    assert r.returncode == 0, (r.stdout + r.stderr)[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["solve"]["status"] == "OK"
    g = json.load(open(os.path.join(HERE, "golden", "oracle_C2.json")))
    assert d["solve"]["a_matvecs_per_solve"] == g["a_matvecs"]
