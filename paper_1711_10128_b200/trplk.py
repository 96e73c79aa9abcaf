"""Thin Python binding of libtrplk.so (include/trplk.h, include/trplk_kernels.h).

Argument marshalling only: every step of TRPL+K runs in the CUDA kernels of the
library.  PyTorch provides device memory (the caching allocator, through the
ABI's trplk_allocator hooks), the stream and the process group used to
broadcast the NCCL unique id.  There is no CPU fallback: if the library is
missing this module raises at import time.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TRPLK_LIB_OVERRIDE") or os.path.join(_PKG, "lib", "libtrplk.so")  # override: A/B tools

if not os.path.exists(LIB_PATH):
    raise ImportError(f"libtrplk.so not built ({LIB_PATH}); run `python -m paper_1711_10128_b200.build`")

_lib = ctypes.CDLL(LIB_PATH)

_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_D = ctypes.c_double
_I = ctypes.c_int

STATUS = {0: "OK", 1: "EINVAL", 2: "NOT_CONVERGED", 3: "BREAKDOWN", 4: "ECUDA", 5: "ENCCL", 6: "ENOMEM"}
MAX_BASIS = 64

_ALLOC_FN = ctypes.CFUNCTYPE(_P, ctypes.c_size_t, _P)
_FREE_FN = ctypes.CFUNCTYPE(None, _P, _P)


class Allocator(ctypes.Structure):
    _fields_ = [("alloc", _ALLOC_FN), ("free", _FREE_FN), ("user", _P)]


class Dist(ctypes.Structure):
    _fields_ = [("rank", _I), ("nranks", _I), ("row_begin", _I64), ("row_end", _I64),
                ("nccl_unique_id", _P)]


_AG_FN = ctypes.CFUNCTYPE(_I, _P, _P, ctypes.c_size_t, _P)
_SR_FN = ctypes.CFUNCTYPE(_I, _I, ctypes.POINTER(_I), ctypes.POINTER(_P), ctypes.POINTER(ctypes.c_size_t),
                          _I, ctypes.POINTER(_I), ctypes.POINTER(_P), ctypes.POINTER(ctypes.c_size_t), _P)
_AR_FN = ctypes.CFUNCTYPE(_I, ctypes.POINTER(_D), _I, _I, _P)


class HostCommS(ctypes.Structure):
    _fields_ = [("allgather", _AG_FN), ("sendrecv", _SR_FN), ("allreduce", _AR_FN), ("user", _P)]


class Options(ctypes.Structure):
    _fields_ = [("seed", ctypes.c_uint64), ("max_cycles", _I), ("tol_mode", _I),
                ("restart_size", _I), ("lock_mode", _I), ("debug_checks", _I), ("use_graphs", _I),
                ("precond", _I), ("block", _I)]


class Stats(ctypes.Structure):
    _fields_ = [("a_matvecs", _I64), ("b_matvecs", _I64), ("precond_applies", _I64),
                ("cycles", _I64), ("inner_steps", _I64), ("verify_matvecs", _I64),
                ("random_draws", _I64), ("status", _I), ("solve_seconds", _D), ("model_bytes", _D),
                ("kernel_launches", _I64)]

    def as_dict(self):
        d = {k: getattr(self, k) for k, _ in self._fields_}
        d["status"] = STATUS.get(d["status"], d["status"])
        return d


def _sig(name, res, args):
    f = getattr(_lib, name)
    f.restype = res
    f.argtypes = args
    return f


_sig("trplk_options_default", None, [ctypes.POINTER(Options)])
_sig("trplk_nccl_unique_id", _I, [_P, ctypes.c_size_t])
_sig("trplk_create", _I, [ctypes.POINTER(_P), _I64, _P, _P, _P, _P, _P, _P, _D,
                          ctypes.POINTER(Dist), ctypes.POINTER(Allocator), _P])
_sig("trplk_solve", _I, [_P, _I, _I, _I, _D, _P, _P, _P, ctypes.POINTER(Options), ctypes.POINTER(Stats)])
_sig("trplk_get_log", _I, [_P, _I, _P, _P, _P, _P, _P, _P, _P])
_sig("trplk_info", _I, [_P, _P, _P, _P, _P, _P, _P, _P])
_sig("trplk_destroy", None, [_P])
_sig("trplk_last_error", ctypes.c_char_p, [_P])
_sig("trplk_k_spmv", _I, [_P, _I, _P, _P])
_sig("trplk_k_step1", _I, [_P, _P, _I64, _I, _P, _D, _P, _P, _P, _P])
_sig("trplk_k_cgs2", _I, [_P, _P, _I64, _I, _P, _P, _P, _P, _P, _P])
_sig("trplk_k_rotate", _I, [_P, _P, _I64, _I, _P, _I, _P, _I64])
_sig("trplk_k_sym_eig", _I, [_P, _I, _P, _P, _P])
_sig("trplk_k_residual", _I, [_P, _P, _D, _P, _P, _P])
_sig("trplk_k_sym_eig_time", _I, [_P, _I, _P, _I, _P, _P])
_sig("trplk_loopback_create", _I, [_I, ctypes.POINTER(_P)])
_sig("trplk_create_ex", _I, [ctypes.POINTER(_P), _I64, _P, _P, _P, _P, _P, _P, _D, _P, _P, _P, _P, _P])
_sig("trplk_set_debug", _I, [_P, _I])
_sig("trplk_loopback_destroy", None, [_P])
_sig("trplk_k_random", _I, [_P, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64, _P])
_sig("trplk_plan_ghosts", _I, [_I64, _I64, _P, _P, _P, _P, _P, _I, _P, _P, _I64, ctypes.POINTER(_I64)])
_sig("trplk_profile", _I, [_P, _I])
_sig("trplk_profile_read", _I, [_P, _P, _P, ctypes.POINTER(_I64)])
_sig("trplk_profile_kernels", _I, [_P, ctypes.c_char_p, ctypes.c_size_t])
_sig("trplk_profile_phases", _I, [_P, _P, ctypes.POINTER(_I64)])
_sig("trplk_k_block", _I, [_P, _I, _P, _I64, _I, _P, _I64, _I, _P, _P, _P, _I64, _P, _P])
_sig("trplk_pl1_solve", _I, [_P, _I, _D, _I, _I, _I, ctypes.c_uint64, _P, _P, _P, _P, _I, _P, _P, _P, _P,
                             ctypes.POINTER(Stats)])
_sig("trplk_pl1_set_qopt", _I, [_P, _I])
_sig("trplk_pl1_get_qopt", _I, [_P, _I, _D, _P, _P, _P])

EXPORTED = ["trplk_options_default", "trplk_nccl_unique_id", "trplk_create", "trplk_solve",
            "trplk_get_log", "trplk_info", "trplk_destroy", "trplk_last_error", "trplk_k_spmv",
            "trplk_k_step1", "trplk_k_cgs2", "trplk_k_rotate", "trplk_k_sym_eig",
            "trplk_k_residual", "trplk_k_random", "trplk_profile", "trplk_profile_read",
            "trplk_plan_ghosts", "trplk_k_sym_eig_time", "trplk_loopback_create", "trplk_loopback_destroy",
            "trplk_set_debug", "trplk_pl1_solve", "trplk_profile_kernels", "trplk_create_ex",
            "trplk_profile_phases", "trplk_k_block", "trplk_pl1_set_qopt", "trplk_pl1_get_qopt"]


class TrplkError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = STATUS.get(status, status)


def _ptr(a):
    if a is None:
        return None
    if hasattr(a, "data_ptr"):
        return a.data_ptr()
    return a.ctypes.data


def _csr_arrays(M):
    if M is None:
        return None, None, None
    if hasattr(M, "rowptr"):
        return (np.ascontiguousarray(M.rowptr, np.int64), np.ascontiguousarray(M.col, np.int64),
                np.ascontiguousarray(M.val, np.float64))
    M = M.tocsr()
    M.sort_indices()
    return (np.ascontiguousarray(M.indptr, np.int64), np.ascontiguousarray(M.indices, np.int64),
            np.ascontiguousarray(M.data, np.float64))


class Context:
    """Owns a trplk_ctx*; created by trplk_create()."""

    def __init__(self, handle, stream, keep):
        self.handle = handle
        self.stream = stream
        self._keep = keep
        n_local, n_ghost, rank, nranks, fro = _I64(), _I64(), _I(), _I(), _D()
        sa, sb = _I64(), _I64()
        _lib.trplk_info(handle, ctypes.byref(n_local), ctypes.byref(n_ghost), ctypes.byref(rank),
                        ctypes.byref(nranks), ctypes.byref(fro), ctypes.byref(sa), ctypes.byref(sb))
        self.n_local, self.n_ghost = n_local.value, n_ghost.value
        self.rank, self.nranks = rank.value, nranks.value
        self.frob_a = fro.value
        self.sell_bytes_a, self.sell_bytes_b = sa.value, sb.value
        self.ld = ((self.n_local + self.n_ghost + 31) // 32) * 32

    def last_error(self) -> str:
        return _lib.trplk_last_error(self.handle).decode()

    def check(self, st):
        if st != 0:
            raise TrplkError(st, self.last_error())

    def close(self):
        if self.handle:
            _lib.trplk_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _torch_allocator(device_index, stream_int):
    import torch

    def _alloc(nbytes, user):
        try:
            return torch.cuda.caching_allocator_alloc(nbytes, device_index, stream_int)
        except Exception:
            return None

    def _free(ptr, user):
        torch.cuda.caching_allocator_delete(ptr)

    fa, ff = _ALLOC_FN(_alloc), _FREE_FN(_free)
    return Allocator(fa, ff, None), (fa, ff)


def trplk_nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    st = _lib.trplk_nccl_unique_id(buf, 128)
    if st != 0:
        raise TrplkError(st, "ncclGetUniqueId failed")
    return buf.raw


def trplk_loopback_create(nranks: int):
    """In-process loopback hub (test infrastructure): ranks of one solve as threads on one GPU."""
    h = _P()
    st = _lib.trplk_loopback_create(int(nranks), ctypes.byref(h))
    if st != 0:
        raise TrplkError(st, "trplk_loopback_create failed")
    return h


def trplk_loopback_destroy(hub):
    _lib.trplk_loopback_destroy(hub)


def trplk_set_debug(ctx, flags: int):
    """Debug switches (bit 0: force the third CGS pass; bit 1: grid-wide cooperative inner loop)."""
    ctx.check(_lib.trplk_set_debug(ctx.handle, int(flags)))


def host_comm(group):
    """trplk_host_comm callbacks over a torch.distributed process group (gloo): the row-partition
    exchanges staged through host memory (several processes may then share one GPU)."""
    import traceback

    import torch
    import torch.distributed as dist

    nr = dist.get_world_size(group)
    grank = (lambda r: dist.get_global_rank(group, r)) if group is not dist.group.WORLD else (lambda r: r)

    def _view(addr, nbytes):
        return torch.from_numpy(np.ctypeslib.as_array((ctypes.c_uint8 * nbytes).from_address(addr)))

    def ag(send, recv, nbytes, user):
        try:
            src = _view(send, nbytes).clone() if nbytes else torch.empty(0, dtype=torch.uint8)
            outs = [torch.empty(nbytes, dtype=torch.uint8) for _ in range(nr)]
            dist.all_gather(outs, src, group=group)
            if nbytes:
                _view(recv, nbytes * nr).copy_(torch.cat(outs))
            return 0
        except Exception:
            traceback.print_exc()
            return 1

    def sr(ns, sp, sb, sn, nrv, rp, rb, rn, user):
        try:
            reqs, bufs = [], []
            for j in range(nrv):
                if rn[j]:
                    t = torch.empty(rn[j], dtype=torch.uint8)
                    bufs.append((t, rb[j], rn[j]))
                    reqs.append(dist.irecv(t, src=grank(rp[j]), group=group))
            for i in range(ns):
                if sn[i]:
                    reqs.append(dist.isend(_view(sb[i], sn[i]).clone(), dst=grank(sp[i]), group=group))
            for q in reqs:
                q.wait()
            for t, addr, nb in bufs:
                _view(addr, nb).copy_(t)
            return 0
        except Exception:
            traceback.print_exc()
            return 1

    def ar(v, count, op, user):
        try:
            t = torch.from_numpy(np.ctypeslib.as_array(v, shape=(count,)).copy())
            dist.all_reduce(t, op=dist.ReduceOp.SUM if op == 0 else dist.ReduceOp.MAX, group=group)
            np.ctypeslib.as_array(v, shape=(count,))[:] = t.numpy()
            return 0
        except Exception:
            traceback.print_exc()
            return 1

    fns = (_AG_FN(ag), _SR_FN(sr), _AR_FN(ar))
    return HostCommS(fns[0], fns[1], fns[2], None), fns


def trplk_create(A, B=None, sigma: float = 0.0, n_global: Optional[int] = None, row_begin: int = 0,
                 row_end: Optional[int] = None, group=None, stream=None, torch_alloc: bool = True,
                 loopback=None, comm: str = "nccl") -> Context:
    """Create a context.  A/B: inputs.CSR (this rank's rows) or scipy CSR.  For several ranks pass
    the torch.distributed `group` and this rank's row range: comm="nccl" (production: rank 0's NCCL
    id is broadcast) or comm="host" (host-staged exchanges through the group's own collectives,
    e.g. gloo; processes may share one GPU).  loopback=(hub, rank, nranks): the rank of an
    in-process loopback solve (tests only)."""
    import torch

    ra, ca, va = _csr_arrays(A)
    rb, cb, vb = _csr_arrays(B)
    if n_global is None:
        n_global = getattr(A, "n", None) or A.shape[1]
    rows = len(ra) - 1
    if row_end is None:
        row_begin = getattr(A, "row_begin", row_begin)
        row_end = row_begin + rows
    dev = torch.cuda.current_device()
    if stream is None:
        stream = torch.cuda.current_stream()
    sptr = stream.cuda_stream
    keep = [ra, ca, va, rb, cb, vb]
    dist_p = None
    hub_p, hc_p = None, None
    if group is not None and comm == "host":
        import torch.distributed as dist
        rank, nranks = dist.get_rank(group), dist.get_world_size(group)
        hc, fns = host_comm(group)
        keep += [hc, fns]
        hc_p = ctypes.byref(hc)
        d = Dist(rank, nranks, row_begin, row_end, None)
        keep.append(d)
        dist_p = ctypes.byref(d)
    elif group is not None:
        import torch.distributed as dist
        rank, nranks = dist.get_rank(group), dist.get_world_size(group)
        idt = torch.zeros(128, dtype=torch.uint8)
        if rank == 0:
            idt[:] = torch.frombuffer(bytearray(trplk_nccl_unique_id()), dtype=torch.uint8)
        if dist.get_backend(group) == "nccl":
            idt = idt.cuda()
        dist.broadcast(idt, src=dist.get_global_rank(group, 0) if hasattr(dist, "get_global_rank") else 0,
                       group=group)
        idb = ctypes.create_string_buffer(bytes(idt.cpu().numpy().tobytes()), 128)
        keep.append(idb)
        d = Dist(rank, nranks, row_begin, row_end, ctypes.cast(idb, _P))
        keep.append(d)
        dist_p = ctypes.byref(d)
    elif loopback is not None:
        hub, rank, nranks = loopback
        d = Dist(rank, nranks, row_begin, row_end, None)
        keep.append(d)
        dist_p = ctypes.byref(d)
        hub_p = hub
    elif row_begin != 0 or row_end != n_global:
        d = Dist(0, 1, row_begin, row_end, None)
        keep.append(d)
        dist_p = ctypes.byref(d)
    alloc_p = None
    if torch_alloc:
        al, fns = _torch_allocator(dev, sptr)
        keep += [al, fns]
        alloc_p = ctypes.byref(al)
    h = _P()
    if hub_p is None and hc_p is None:
        st = _lib.trplk_create(ctypes.byref(h), n_global, _ptr(ra), _ptr(ca), _ptr(va), _ptr(rb), _ptr(cb),
                               _ptr(vb), float(sigma), dist_p, alloc_p, sptr)
    else:
        st = _lib.trplk_create_ex(ctypes.byref(h), n_global, _ptr(ra), _ptr(ca), _ptr(va), _ptr(rb), _ptr(cb),
                                  _ptr(vb), float(sigma), dist_p, hub_p, hc_p, alloc_p, sptr)
    if st != 0:
        msg = _lib.trplk_last_error(h).decode() if h.value else "create failed"
        if h.value:
            _lib.trplk_destroy(h)
        raise TrplkError(st, msg)
    return Context(h, stream, keep)


def make_options(**kw) -> Options:
    o = Options()
    _lib.trplk_options_default(ctypes.byref(o))
    for k, v in kw.items():
        if not hasattr(o, k):
            raise TypeError(f"unknown option {k}")
        setattr(o, k, v)
    return o


def trplk_solve(ctx: Context, p: int, max_basis: int, k_plus: int, tol: float, evecs_out=None,
                **options):
    """Run Algorithm 1.  Returns (eigenvalues np[p], eigenvectors torch.cuda (n_local, p)
    column-major view, residual norms np[p], stats dict).  Raises on error statuses except
    NOT_CONVERGED / BREAKDOWN (reported in stats['status'])."""
    import torch

    opt = make_options(**options)
    ev = np.zeros(p)
    rs = np.zeros(p)
    if evecs_out is None:
        buf = torch.empty((p, ctx.n_local), dtype=torch.float64, device="cuda")
        evecs = buf.T
        ptr = buf.data_ptr()
    else:
        evecs = evecs_out
        ptr = _ptr(evecs_out)
    stats = Stats()
    st = _lib.trplk_solve(ctx.handle, p, max_basis, k_plus, tol, _ptr(ev), ptr, _ptr(rs), ctypes.byref(opt),
                          ctypes.byref(stats))
    if st not in (0, 2, 3):
        ctx.check(st)
    return ev, evecs, rs, stats.as_dict()


def trplk_pl1_solve(ctx: Context, m: int, tol: float, variant: int = 0, use_precond: bool = True,
                    max_iter: int = 2000, seed: int = 12, x0=None, x_out=None):
    """PL+1 (Algorithm 2) for the lowest eigenpair.  Returns (rho, residual, x torch.cuda (n_local,)
    or x_out, stats dict, log dict {rho, res, conj})."""
    import torch

    x = torch.empty(ctx.n_local, dtype=torch.float64, device="cuda") if x_out is None else x_out
    cap = int(max_iter) + 1
    lr, ls, lc = np.zeros(cap), np.zeros(cap), np.zeros(cap)
    nlog = _I(0)
    rho, res = _D(0.0), _D(0.0)
    stats = Stats()
    x0p = None
    if x0 is not None:
        x0 = np.ascontiguousarray(x0, np.float64) if not hasattr(x0, "data_ptr") else x0
        x0p = _ptr(x0)
    st = _lib.trplk_pl1_solve(ctx.handle, int(m), float(tol), int(variant), 1 if use_precond else 0, int(max_iter),
                              int(seed), x0p, ctypes.byref(rho), ctypes.byref(res), _ptr(x), cap, _ptr(lr),
                              _ptr(ls), _ptr(lc), ctypes.byref(nlog), ctypes.byref(stats))
    if st not in (0, 2, 3):
        ctx.check(st)
    L = nlog.value
    return rho.value, res.value, x, stats.as_dict(), {"rho": lr[:L], "res": ls[:L], "conj": lc[:L]}


def trplk_pl1_set_qopt(ctx: Context, cap: int):
    """Arm (cap > 0, <= 64) or disarm (0) the PL+1 quasi-optimality diagnostic (reading P7)."""
    ctx.check(_lib.trplk_pl1_set_qopt(ctx.handle, int(cap)))


def trplk_pl1_get_qopt(ctx: Context, cap: int = 64, lambda1: float = float("nan")):
    """Of the last PL+1 solve: {rho_star, dim, ratio} per iteration (entry k = U_k)."""
    rs, dm, ra = np.zeros(cap), np.zeros(cap, np.int32), np.zeros(cap)
    L = _lib.trplk_pl1_get_qopt(ctx.handle, int(cap), float(lambda1), _ptr(rs), _ptr(dm), _ptr(ra))
    return {"rho_star": rs[:L], "dim": dm[:L], "ratio": ra[:L]}


def trplk_get_log(ctx: Context, cap: int = 100000, ph: Optional[int] = None):
    cap = int(cap)
    t = np.zeros(cap, np.int32)
    mv = np.zeros(cap, np.int64)
    th = np.zeros(cap)
    rs = np.zeros(cap)
    k = np.zeros(cap, np.int32)
    npv = np.zeros(cap, np.int32)
    ths = np.zeros((cap, ph)) if ph else None
    n = _lib.trplk_get_log(ctx.handle, cap, _ptr(t), _ptr(mv), _ptr(th), _ptr(rs), _ptr(k), _ptr(npv),
                           _ptr(ths))
    out = {"t": t[:n], "mv": mv[:n], "theta_t": th[:n], "res": rs[:n], "k": k[:n], "nprev": npv[:n]}
    if ph:
        out["thetas"] = ths[:n]
    return out


def trplk_destroy(ctx: Context):
    ctx.close()


def trplk_last_error(ctx: Context) -> str:
    return ctx.last_error()


# ------------------------------------------------------------ kernel-level entry points
def trplk_k_spmv(ctx, which, x, y):
    ctx.check(_lib.trplk_k_spmv(ctx.handle, which, _ptr(x), _ptr(y)))


def trplk_k_step1(ctx, U, ldu, k, g, rho, w):
    tcol, h1, nrm = np.zeros(k), np.zeros(k), _D()
    ctx.check(_lib.trplk_k_step1(ctx.handle, _ptr(U), ldu, k, _ptr(g), rho, _ptr(w), _ptr(tcol), _ptr(h1),
                                 ctypes.byref(nrm)))
    return tcol, h1, nrm.value


def trplk_k_cgs2(ctx, U, ldu, k, w, out):
    h = np.zeros(max(k, 1))
    beta, brk, passes = _D(), _I(), _I()
    ctx.check(_lib.trplk_k_cgs2(ctx.handle, _ptr(U), ldu, k, _ptr(w), _ptr(out), _ptr(h), ctypes.byref(beta),
                                ctypes.byref(brk), ctypes.byref(passes)))
    return h[:k], beta.value, bool(brk.value), passes.value


def trplk_k_rotate(ctx, U, ldu, k, Y, ncol, X, ldx):
    Y = np.asfortranarray(Y, np.float64)
    ctx.check(_lib.trplk_k_rotate(ctx.handle, _ptr(U), ldu, k, _ptr(Y), ncol, _ptr(X), ldx))


def trplk_k_sym_eig(ctx, T):
    T = np.asfortranarray(T, np.float64)
    k = T.shape[0]
    th = np.zeros(k)
    Y = np.zeros((k, k), order="F")
    ctx.check(_lib.trplk_k_sym_eig(ctx.handle, k, _ptr(T), _ptr(th), _ptr(Y)))
    return th, Y


def trplk_k_sym_eig_time(ctx, T, reps=50):
    """Average device ms per launch of the Rayleigh-Ritz kernel on sym(T), and its sweep count."""
    T = np.asfortranarray(T, np.float64)
    ms = _D()
    sw = ctypes.c_int()
    ctx.check(_lib.trplk_k_sym_eig_time(ctx.handle, T.shape[0], _ptr(T), int(reps), ctypes.byref(ms),
                                        ctypes.byref(sw)))
    return ms.value, sw.value


def trplk_k_residual(ctx, x, theta, r=None, u=None):
    n2 = _D()
    ctx.check(_lib.trplk_k_residual(ctx.handle, _ptr(x), theta, _ptr(r), _ptr(u), ctypes.byref(n2)))
    return n2.value


def trplk_k_random(ctx, seed, stream, col, x):
    ctx.check(_lib.trplk_k_random(ctx.handle, seed, stream, col, _ptr(x)))


def trplk_options_default() -> Options:
    return make_options()


def trplk_info(ctx: Context) -> dict:
    return {"n_local": ctx.n_local, "n_ghost": ctx.n_ghost, "rank": ctx.rank, "nranks": ctx.nranks,
            "frob_a": ctx.frob_a, "sell_bytes_a": ctx.sell_bytes_a, "sell_bytes_b": ctx.sell_bytes_b}


def trplk_plan_ghosts(A, B=None, row_begin=0, row_end=None, ranges=None):
    """Host-only halo plan of a row slab (the code trplk_create runs): (ghost ids, owner ranks)."""
    ra, ca, _ = _csr_arrays(A)
    rb, cb, _ = _csr_arrays(B)
    if row_end is None:
        row_end = row_begin + len(ra) - 1
    rg = None if ranges is None else np.ascontiguousarray(np.asarray(ranges, np.int64).ravel())
    nr = 1 if rg is None else len(rg) // 2
    cnt = _I64()
    _lib.trplk_plan_ghosts(row_begin, row_end, _ptr(ra), _ptr(ca), _ptr(rb), _ptr(cb), _ptr(rg), nr, None,
                           None, 0, ctypes.byref(cnt))
    g = np.zeros(max(cnt.value, 1), np.int64)
    o = np.zeros(max(cnt.value, 1), np.int32)
    st = _lib.trplk_plan_ghosts(row_begin, row_end, _ptr(ra), _ptr(ca), _ptr(rb), _ptr(cb), _ptr(rg), nr,
                                _ptr(g), _ptr(o), len(g), ctypes.byref(cnt))
    if st != 0:
        raise TrplkError(st, "trplk_plan_ghosts failed")
    return g[:cnt.value], o[:cnt.value]


def trplk_profile(ctx: Context, enable: bool = True):
    ctx.check(_lib.trplk_profile(ctx.handle, 1 if enable else 0))


def trplk_profile_read(ctx: Context) -> dict:
    """Accumulated live inner-step profile: per kernel group (K1, K2, K3) the device ms and
    algorithmic bytes summed over `count` cycles."""
    ms = np.zeros(3)
    by = np.zeros(3)
    cnt = _I64()
    ctx.check(_lib.trplk_profile_read(ctx.handle, _ptr(ms), _ptr(by), ctypes.byref(cnt)))
    return {"ms": ms, "bytes": by, "count": cnt.value}


def trplk_profile_kernels(ctx: Context) -> list:
    """Names of the kernel instantiations that ran the profiled groups K1, K2, K3 ('' where a
    group is fused into K1), as the library launched them (demangled)."""
    buf = ctypes.create_string_buffer(4096)
    ctx.check(_lib.trplk_profile_kernels(ctx.handle, buf, len(buf)))
    return buf.value.decode().split(";")


def trplk_create_ex(A, B=None, sigma: float = 0.0, **kw) -> Context:
    """trplk_create with the exchanges through a loopback hub (loopback=(hub, rank, nranks)) or a
    host-staged process group (group=..., comm="host"): the C entry trplk_create_ex."""
    if kw.get("loopback") is None and kw.get("comm", "nccl") != "host":
        raise TypeError("trplk_create_ex needs loopback=(hub, rank, nranks) or group=..., comm='host'")
    return trplk_create(A, B, sigma, **kw)


PHASES = ["seed CGS2", "inner steps", "+K", "RR eig", "rotation", "residual"]


def trplk_profile_phases(ctx: Context) -> dict:
    """Live cycle-phase profile: device ms per phase summed over `count` profiled cycles."""
    ms = np.zeros(6)
    cnt = _I64()
    ctx.check(_lib.trplk_profile_phases(ctx.handle, _ptr(ms), ctypes.byref(cnt)))
    return {"phases": PHASES, "ms": ms, "count": cnt.value}


def trplk_k_block(ctx, mode, U, ldu, k, Y, ldy, c, Rinv=None, H=None, Yout=None, ldyo=0):
    """Block kernel (mode 0 GRAM, 1 UPD, 2 SPMM) on device blocks U (k columns) and Y (c columns);
    returns (HV k x c, G c x c) as numpy arrays."""
    HV = np.zeros((k, c), order="F")
    G = np.zeros((c, c), order="F")
    R = None if Rinv is None else np.asfortranarray(Rinv, np.float64)
    Hh = None if H is None else np.asfortranarray(H, np.float64)
    ctx.check(_lib.trplk_k_block(ctx.handle, int(mode), _ptr(U), ldu, k, _ptr(Y), ldy, c, _ptr(R), _ptr(Hh),
                                 _ptr(Yout), ldyo, _ptr(HV), _ptr(G)))
    return HV, G
