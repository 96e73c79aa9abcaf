"""World-size-2 CPU tests (gloo) of the multi-GPU host logic: z-slab row
partition, ghost discovery and owner assignment (trplk_plan_ghosts = the code trplk_create
runs), the halo exchange plan, the local column remapping, and the deterministic
allgather-then-fixed-order-sum reduction used for every dot product across ranks."""
import os
import socket

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, cfg, N, q):
    import sys
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1711_10128_b200 import inputs, trplk
        full = inputs.make(cfg, N=N)
        n = full.A.n
        plane = 1 if full.grid["dim"] == 1 else N * N
        rb, re = inputs.slab_rows(n, world, rank, plane)
        P = inputs.make(cfg, N=N, row_begin=rb, row_end=re)
        ranges = [None] * world
        dist.all_gather_object(ranges, (rb, re))
        assert ranges[0][0] == 0 and ranges[-1][1] == n
        assert all(ranges[r][1] == ranges[r + 1][0] for r in range(world - 1))
        ghosts, owners = trplk.trplk_plan_ghosts(P.A, P.B, rb, re, np.array(ranges))
        # ghosts: outside the slab, owned by the rank whose range contains them, contiguous planes
        for g, o in zip(ghosts, owners):
            assert not (rb <= g < re)
            assert ranges[o][0] <= g < ranges[o][1]
        lo = ghosts[ghosts < rb]
        hi = ghosts[ghosts >= re]
        if len(lo):
            assert np.array_equal(lo, np.arange(rb - len(lo), rb))  # DIA-eligible halo
        if len(hi):
            assert np.array_equal(hi, np.arange(re, re + len(hi)))
        # halo exchange plan: every rank requests its ghosts from their owners
        reqs = [None] * world
        dist.all_gather_object(reqs, (ghosts.tolist(), owners.tolist()))
        x = inputs.u01(12, 0, 0, n)  # the global vector, seeded (each rank sends its own rows only)
        send = {}
        for r2 in range(world):
            if r2 == rank:
                continue
            gl, ow = reqs[r2]
            ids = [g for g, o in zip(gl, ow) if o == rank]
            send[r2] = x[np.array(ids, dtype=np.int64)] if ids else np.zeros(0)
        recv = [None] * world
        dist.all_gather_object(recv, send)
        ghost_vals = np.zeros(len(ghosts))
        for i, (g, o) in enumerate(zip(ghosts, owners)):
            gl_o = [gg for gg, oo in zip(*reqs[rank]) if oo == o]
            ghost_vals[i] = recv[o][rank][gl_o.index(g)]
        x_ext = np.concatenate([x[rb:re], ghost_vals])
        # local column remapping (trplk.h: owned c - row_begin, ghost n_local + index)
        nl = re - rb
        for M, Mf in ((P.A, full.A), (P.B, full.B)):
            if M is None:
                continue
            loc = np.where((M.col >= rb) & (M.col < re), M.col - rb, nl + np.searchsorted(ghosts, M.col))
            y_loc = np.array([np.dot(M.val[M.rowptr[i]:M.rowptr[i + 1]], x_ext[loc[M.rowptr[i]:M.rowptr[i + 1]]])
                              for i in range(nl)])
            y_glob = Mf.to_scipy() @ x
            assert np.allclose(y_loc, y_glob[rb:re], rtol=1e-15, atol=1e-14)
        # deterministic cross-rank reduction: allgather of per-rank partials + fixed-order sum
        k = 6
        U = np.stack([inputs.u01(12, 0, c * n, n) for c in range(k)], axis=1)
        part = U[rb:re].T @ x[rb:re]
        parts = [None] * world
        dist.all_gather_object(parts, part)
        tot = parts[0].copy()
        for r2 in range(1, world):
            tot = tot + parts[r2]
        mine = [None] * world
        dist.all_gather_object(mine, tot.tobytes())
        assert all(m == mine[0] for m in mine)  # bitwise identical on every rank
        assert np.allclose(tot, U.T @ x, rtol=1e-13)
        q.put((rank, "ok", len(ghosts)))
    except Exception as e:  # pragma: no cover - reported to the parent
        import traceback
        q.put((rank, "fail", traceback.format_exc()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("cfg,N", [("C2", 8), ("C4", 6), ("C1", None)])
def test_slab_partition_world2(cfg, N):
    import torch.multiprocessing as mp
    from paper_1711_10128_b200 import build
    build.build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    N_ = N if N is not None else 1000
    procs = [ctx.Process(target=_worker, args=(r, 2, port, cfg, N_, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for r in res:
        assert r[1] == "ok", r
    assert all(r[2] > 0 for r in res)  # each slab has a halo


def _hostcomm_worker(rank, world, port, q):
    """The host-staged exchange callbacks (trplk.host_comm: what trplk_create_ex calls for
    comm='host') over a world-size-2 gloo group, called through their C function pointers exactly
    as the library calls them: allgather in rank order, grouped send/recv with per-peer sizes, and
    the create-time sum / max allreduce."""
    import ctypes
    import sys
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1711_10128_b200 import trplk
        hc, fns = trplk.host_comm(dist.group.WORLD)
        # allgather: 5 doubles per rank -> rank-ordered concatenation
        send = np.arange(5, dtype=np.float64) + 100 * rank
        recv = np.zeros(5 * world)
        assert hc.allgather(send.ctypes.data, recv.ctypes.data, send.nbytes, None) == 0
        assert np.array_equal(recv, np.concatenate([np.arange(5) + 100 * r for r in range(world)]))
        # sendrecv: a halo-like exchange with different sizes per direction (int64 and fp64 payloads)
        peer = 1 - rank
        out = np.arange(3 + rank, dtype=np.int64) * (rank + 1)
        inn = np.zeros(3 + peer, dtype=np.int64)
        sp = (ctypes.c_int * 1)(peer)
        sb = (ctypes.c_void_p * 1)(out.ctypes.data)
        sn = (ctypes.c_size_t * 1)(out.nbytes)
        rb_ = (ctypes.c_void_p * 1)(inn.ctypes.data)
        rn = (ctypes.c_size_t * 1)(inn.nbytes)
        assert hc.sendrecv(1, sp, sb, sn, 1, sp, rb_, rn, None) == 0
        assert np.array_equal(inn, np.arange(3 + peer) * (peer + 1))
        # allreduce: sum and max of host doubles (create: ||A||_F^2, max |A_jj|)
        v = np.array([1.5 + rank, -2.0 * rank])
        assert hc.allreduce(v.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), 2, 0, None) == 0
        assert np.array_equal(v, [1.5 + 2.5, -2.0])
        w = np.array([3.0 * rank, 7.0 - rank])
        assert hc.allreduce(w.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), 2, 1, None) == 0
        assert np.array_equal(w, [3.0, 7.0])
        q.put((rank, "ok", None))
    except Exception:  # pragma: no cover - reported to the parent
        import traceback
        q.put((rank, "fail", traceback.format_exc()))
    finally:
        dist.destroy_process_group()


def test_host_comm_callbacks_world2():
    import torch.multiprocessing as mp
    from paper_1711_10128_b200 import build
    build.build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_hostcomm_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for r in res:
        assert r[1] == "ok", r
