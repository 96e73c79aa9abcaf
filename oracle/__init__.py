"""TRPL+K CPU oracle -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` leg may import this package.  It wraps ``oracle.c`` (plain
fp64 C + OpenMP, Algorithm 1 of PAPER.md:176-202 with the readings of
DESIGN.md) via ctypes.  It shares no code with ``paper_1711_10128_b200``.

Pins (tests/test_oracle_*.py): closed-form Laplacian spectra, dense
``numpy.linalg.eigh`` / ``scipy.linalg.eigh(A, B)`` brute force on tiny
problems, analytic sine eigenvectors for SpMV, ``math.fsum`` for dots, B-
orthonormality, eq 3.1 bookkeeping, cross-cycle interlacing, the eq 3.2
subspace rebuilt densely, LOPCG and TRLan reductions, exact matvec accounting.
Parity unpinned: the matvec count to convergence (no paper value for these
synthetic matrices; SURVEY 8(c.4) last row).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_HDR = os.path.join(_HERE, "oracle.h")
_LIB = os.path.join(_HERE, "liboracle.so")

_P = ctypes.c_void_p
_I64 = ctypes.c_int64


def build(force: bool = False) -> str:
    newest = max(os.path.getmtime(_SRC), os.path.getmtime(_HDR))
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < newest:
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c11",
                               "-o", _LIB, _SRC, "-lm"])
    return _LIB


class _Problem(ctypes.Structure):
    _fields_ = [("n", _I64), ("a_rowptr", _P), ("a_col", _P), ("a_val", _P),
                ("b_rowptr", _P), ("b_col", _P), ("b_val", _P), ("sigma", ctypes.c_double),
                ("p", ctypes.c_int), ("q", ctypes.c_int), ("l", ctypes.c_int),
                ("tol", ctypes.c_double), ("tol_mode", ctypes.c_int), ("seed", ctypes.c_uint64),
                ("max_cycles", ctypes.c_int), ("restart_size", ctypes.c_int),
                ("lock_mode", ctypes.c_int), ("debug", ctypes.c_int), ("precond", ctypes.c_int),
                ("block", ctypes.c_int)]


class _Report(ctypes.Structure):
    _fields_ = [("status", ctypes.c_int), ("cycles", ctypes.c_int),
                ("a_matvecs", _I64), ("b_matvecs", _I64), ("precond_applies", _I64),
                ("verify_matvecs", _I64), ("inner_steps", _I64), ("random_draws", _I64),
                ("log_cap", ctypes.c_int), ("log_len", ctypes.c_int),
                ("log_t", _P), ("log_mv", _P), ("log_theta_t", _P), ("log_res", _P),
                ("log_k", _P), ("log_nprev", _P), ("log_thetas", _P), ("log_terr", _P),
                ("log_orth", _P), ("dump_cycles", ctypes.c_int), ("dump_X", _P),
                ("dump_rho", _P), ("dump_t", _P), ("n_sample", ctypes.c_int),
                ("sample_rows", _P), ("sample_vals", _P), ("verbose", ctypes.c_int)]


class _Pl1Problem(ctypes.Structure):
    _fields_ = [("n", _I64), ("a_rowptr", _P), ("a_col", _P), ("a_val", _P),
                ("b_rowptr", _P), ("b_col", _P), ("b_val", _P), ("sigma", ctypes.c_double),
                ("use_precond", ctypes.c_int), ("m", ctypes.c_int), ("tol", ctypes.c_double),
                ("seed", ctypes.c_uint64), ("x0", _P), ("max_cycles", ctypes.c_int),
                ("variant", ctypes.c_int)]


class _Pl1Report(ctypes.Structure):
    _fields_ = [("status", ctypes.c_int), ("cycles", ctypes.c_int),
                ("a_matvecs", _I64), ("b_matvecs", _I64),
                ("rho", ctypes.c_double), ("resid", ctypes.c_double),
                ("log_cap", ctypes.c_int), ("log_len", ctypes.c_int),
                ("log_rho", _P), ("log_res", _P), ("log_conj", _P), ("log_ritz", _P),
                ("log_mg", _P), ("log_nq", _P),
                ("qopt_cap", ctypes.c_int), ("log_qopt", _P), ("log_qdim", _P), ("log_g", _P)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        L.orc_u01.restype = ctypes.c_double
        L.orc_u01.argtypes = [ctypes.c_uint64] * 3
        L.orc_spmv.restype = None
        L.orc_spmv.argtypes = [_I64, _P, _P, _P, _P, _P]
        L.orc_dot.restype = ctypes.c_double
        L.orc_dot.argtypes = [_I64, _P, _P]
        L.orc_frobenius.restype = ctypes.c_double
        L.orc_frobenius.argtypes = [_I64, _P]
        L.orc_jacobi_diag.restype = None
        L.orc_jacobi_diag.argtypes = [_I64, _P, _P, _P, _P, _P, _P, ctypes.c_double,
                                      ctypes.c_double, _P]
        L.orc_sym_eig.restype = ctypes.c_int
        L.orc_sym_eig.argtypes = [ctypes.c_int, _P, _P, _P]
        L.orc_cgs2.restype = ctypes.c_int
        L.orc_cgs2.argtypes = [_I64, ctypes.c_int, _P, _P, _P, _P, _P, _P, _P, _P]
        L.orc_rotate.restype = None
        L.orc_rotate.argtypes = [_I64, ctypes.c_int, _P, _P, ctypes.c_int, ctypes.c_int, _P]
        L.orc_trplk_solve.restype = ctypes.c_int
        L.orc_trplk_solve.argtypes = [ctypes.POINTER(_Problem), _P, _P, _P, ctypes.POINTER(_Report)]
        L.orc_inner_steps.restype = ctypes.c_int
        L.orc_inner_steps.argtypes = [ctypes.POINTER(_Problem), _P, ctypes.c_double, _P, ctypes.c_int,
                                      ctypes.c_int, _P, ctypes.c_int, _P]
        L.orc_ic0.restype = _I64
        L.orc_ic0.argtypes = [ctypes.POINTER(_Problem), ctypes.c_double, _P, _P, _P, _I64]
        L.orc_pl1_solve.restype = ctypes.c_int
        L.orc_pl1_solve.argtypes = [ctypes.POINTER(_Pl1Problem), _P, ctypes.POINTER(_Pl1Report)]
        _lib = L
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data


def _csr(M):
    """Accept inputs.CSR or scipy.sparse csr; return (rowptr int64, col int64, val f64)."""
    if M is None:
        return None, None, None
    if hasattr(M, "rowptr"):
        return (np.ascontiguousarray(M.rowptr, np.int64), np.ascontiguousarray(M.col, np.int64),
                np.ascontiguousarray(M.val, np.float64))
    M = M.tocsr()
    M.sort_indices()
    return (np.ascontiguousarray(M.indptr, np.int64), np.ascontiguousarray(M.indices, np.int64),
            np.ascontiguousarray(M.data, np.float64))


def u01(seed, stream, index):
    return lib().orc_u01(seed, stream, index)


def spmv(A, x):
    rp, ci, v = _csr(A)
    x = np.ascontiguousarray(x, np.float64)
    n = len(rp) - 1
    y = np.empty(n, np.float64)
    lib().orc_spmv(n, _ptr(rp), _ptr(ci), _ptr(v), _ptr(x), _ptr(y))
    return y


def dot(x, y):
    x = np.ascontiguousarray(x, np.float64)
    y = np.ascontiguousarray(y, np.float64)
    return lib().orc_dot(len(x), _ptr(x), _ptr(y))


def frobenius(A):
    _, _, v = _csr(A)
    return lib().orc_frobenius(len(v), _ptr(v))


def jacobi_diag(A, B=None, sigma=0.0, floor_rel=1e-8):
    ra, ca, va = _csr(A)
    rb, cb, vb = _csr(B)
    n = len(ra) - 1
    M = np.empty(n, np.float64)
    lib().orc_jacobi_diag(n, _ptr(ra), _ptr(ca), _ptr(va), _ptr(rb), _ptr(cb), _ptr(vb),
                          sigma, floor_rel, _ptr(M))
    return M


def sym_eig(T):
    T = np.asfortranarray(T, np.float64)
    k = T.shape[0]
    th = np.empty(k, np.float64)
    Y = np.empty((k, k), np.float64, order="F")
    sweeps = lib().orc_sym_eig(k, _ptr(T), _ptr(th), _ptr(Y))
    if sweeps < 0:
        raise RuntimeError("oracle Jacobi did not converge")
    return th, Y


def rotate(U, Y):
    """X = U Y (n x k times k x ncol), column-major fp64."""
    U = np.asfortranarray(U, np.float64)
    Y = np.asfortranarray(Y, np.float64)
    n, k = U.shape
    ncol = Y.shape[1]
    X = np.zeros((n, ncol), order="F")
    lib().orc_rotate(n, k, _ptr(U), _ptr(Y), Y.shape[0], ncol, _ptr(X))
    return X


def cgs2(V, w, B=None):
    """Returns (w_out unnormalised, h (summed coefficients), beta, breakdown, passes)."""
    V = np.asfortranarray(V, np.float64)
    n, k = V.shape
    w = np.array(w, dtype=np.float64, copy=True)
    rb, cb, vb = _csr(B)
    h = np.empty(max(k, 1), np.float64)
    beta = ctypes.c_double()
    passes = ctypes.c_int()
    brk = lib().orc_cgs2(n, k, _ptr(V), _ptr(w), _ptr(rb), _ptr(cb), _ptr(vb), _ptr(h),
                         ctypes.addressof(beta), ctypes.addressof(passes))
    return w, h[:k], beta.value, bool(brk), passes.value


STATUS = {0: "OK", 1: "EINVAL", 2: "NOT_CONVERGED", 3: "BREAKDOWN"}


def solve(A, B=None, p=5, q=20, l=1, tol=1e-8, sigma=0.0, seed=12, max_cycles=5000,
          tol_mode=0, restart_size=0, lock_mode=0, debug=False, dump_cycles=0,
          want_vectors=True, sample_rows=None, verbose=False, precond=0, block=1):
    """Run Algorithm 1 (TRPL+K).  Returns a dict with eigenvalues, vectors, residuals,
    counters and the per-cycle log."""
    ra, ca, va = _csr(A)
    rb, cb, vb = _csr(B)
    n = len(ra) - 1
    ph = restart_size if restart_size > 0 else p
    prob = _Problem(n, _ptr(ra), _ptr(ca), _ptr(va), _ptr(rb), _ptr(cb), _ptr(vb), sigma,
                    p, q, l, tol, tol_mode, seed, max_cycles, restart_size, lock_mode,
                    1 if debug else 0, precond, block)
    cap = max_cycles
    logs = {
        "t": np.zeros(cap, np.int32), "mv": np.zeros(cap, np.int64),
        "theta_t": np.zeros(cap), "res": np.zeros(cap), "k": np.zeros(cap, np.int32),
        "nprev": np.zeros(cap, np.int32), "thetas": np.zeros((cap, ph)),
        "terr": np.zeros(cap), "orth": np.zeros(cap),
    }
    dX = np.zeros((max(dump_cycles, 1), ph, n)) if dump_cycles else None
    drho = np.zeros(max(dump_cycles, 1))
    dt = np.zeros(max(dump_cycles, 1), np.int32)
    srows = None if sample_rows is None else np.ascontiguousarray(sample_rows, np.int64)
    svals = None if srows is None else np.zeros((p, len(srows)))
    rep = _Report(0, 0, 0, 0, 0, 0, 0, 0, cap, 0,
                  _ptr(logs["t"]), _ptr(logs["mv"]), _ptr(logs["theta_t"]), _ptr(logs["res"]),
                  _ptr(logs["k"]), _ptr(logs["nprev"]), _ptr(logs["thetas"]), _ptr(logs["terr"]),
                  _ptr(logs["orth"]), dump_cycles, _ptr(dX), _ptr(drho), _ptr(dt),
                  0 if srows is None else len(srows), _ptr(srows), _ptr(svals), 1 if verbose else 0)
    evals = np.zeros(p)
    resid = np.zeros(p)
    evecs = np.zeros((p, n)) if want_vectors else None  # row c = eigenvector c (n contiguous)
    st = lib().orc_trplk_solve(ctypes.byref(prob), _ptr(evals), _ptr(evecs), _ptr(resid),
                               ctypes.byref(rep))
    L = rep.log_len
    out = {
        "status": STATUS.get(st, st), "eigenvalues": evals, "residuals": resid,
        "eigenvectors": None if evecs is None else evecs.T,
        "cycles": rep.cycles, "a_matvecs": rep.a_matvecs, "b_matvecs": rep.b_matvecs,
        "precond_applies": rep.precond_applies, "verify_matvecs": rep.verify_matvecs,
        "inner_steps": rep.inner_steps, "random_draws": rep.random_draws,
        "log": {k_: v[:L] for k_, v in logs.items()},
        "samples": None if svals is None else svals.T,  # [n_sample, p]
    }
    if dump_cycles:
        nd = min(dump_cycles, rep.cycles)
        out["dump"] = {"X": [dX[i].T.copy() for i in range(nd)], "rho": drho[:nd].copy(),
                       "t": dt[:nd].copy()}
    return out


def inner_steps(A, B, M, rho, U, k0, nsteps, T=None, work=None):
    """Run `nsteps` inner steps of eq 3.1 (orc_inner_steps) on the Fortran-ordered basis U
    (n x (k0+nsteps), orthonormal first k0 columns); fills U's next columns and T in place.
    work: optional scratch of 4n doubles (pre-touched by the caller)."""
    ra, ca, va = _csr(A)
    rb, cb, vb = _csr(B)
    n = len(ra) - 1
    assert U.flags["F_CONTIGUOUS"] and U.dtype == np.float64 and U.shape[1] >= k0 + nsteps
    q = U.shape[1]
    T = np.zeros((q, q), order="F") if T is None else T
    prob = _Problem(n, _ptr(ra), _ptr(ca), _ptr(va), _ptr(rb), _ptr(cb), _ptr(vb), 0.0,
                    1, q, 0, 1.0, 0, 12, 1, 0, 0, 0, 0, 1)
    M = np.ascontiguousarray(M, np.float64)
    if work is not None:
        assert work.dtype == np.float64 and work.size >= 4 * n and work.flags["C_CONTIGUOUS"]
    done = lib().orc_inner_steps(ctypes.byref(prob), _ptr(M), float(rho), _ptr(U), k0, nsteps, _ptr(T), q,
                                 _ptr(work))
    return done, T


def ic0(A, B=None, sigma=0.0):
    """IC(0) factor of A - sigma B (orc_ic0) as a scipy CSR lower-triangular matrix."""
    import scipy.sparse as sp
    ra, ca, va = _csr(A)
    rb, cb, vb = _csr(B)
    n = len(ra) - 1
    prob = _Problem(n, _ptr(ra), _ptr(ca), _ptr(va), _ptr(rb), _ptr(cb), _ptr(vb), sigma,
                    1, 2, 0, 1.0, 0, 12, 1, 0, 0, 0, 3, 1)
    nnz = lib().orc_ic0(ctypes.byref(prob), sigma, None, None, None, 0)
    rp = np.zeros(n + 1, np.int64)
    ci = np.zeros(nnz, np.int64)
    v = np.zeros(nnz)
    lib().orc_ic0(ctypes.byref(prob), sigma, _ptr(rp), _ptr(ci), _ptr(v), nnz)
    return sp.csr_matrix((v, ci, rp), shape=(n, n))


def pl1_solve(A, B=None, m=4, tol=1e-8, sigma=0.0, seed=12, x0=None, max_cycles=2000, variant=0,
              use_precond=True, qopt_cap=0, want_g=False):
    """Run Algorithm 2 (PL+1) for the lowest eigenpair of (A, B), readings P1-P6.  Returns a dict
    with rho, x (B-normalised), residual norm, counters and the per-iteration log.  qopt_cap > 0:
    also the quasi-optimality diagnostic (P7, Def. defnglbopt) in log["qopt"]
    (rho(y*_k) over U_k) and log["qdim"] (dim U_k) for k < qopt_cap; want_g: g_k in "g" (n x cap)."""
    ra, ca, va = _csr(A)
    rb, cb, vb = _csr(B)
    n = len(ra) - 1
    x0a = None if x0 is None else np.ascontiguousarray(x0, np.float64)
    prob = _Pl1Problem(n, _ptr(ra), _ptr(ca), _ptr(va), _ptr(rb), _ptr(cb), _ptr(vb), sigma,
                       1 if use_precond else 0, m, tol, seed, _ptr(x0a), max_cycles, variant)
    cap = max_cycles + 1
    logs = {"rho": np.zeros(cap), "res": np.zeros(cap), "conj": np.zeros(cap), "ritz": np.zeros(cap),
            "mg": np.zeros(cap, np.int32), "nq": np.zeros(cap, np.int32)}
    qo = np.zeros(max(qopt_cap, 1))
    qd = np.zeros(max(qopt_cap, 1), np.int32)
    gl = np.zeros((max(qopt_cap, 1), n)) if (want_g and qopt_cap > 0) else None
    rep = _Pl1Report(0, 0, 0, 0, 0.0, 0.0, cap, 0, _ptr(logs["rho"]), _ptr(logs["res"]),
                     _ptr(logs["conj"]), _ptr(logs["ritz"]), _ptr(logs["mg"]), _ptr(logs["nq"]),
                     qopt_cap, _ptr(qo), _ptr(qd), _ptr(gl))
    x = np.zeros(n)
    st = lib().orc_pl1_solve(ctypes.byref(prob), _ptr(x), ctypes.byref(rep))
    L = rep.log_len
    out = {"status": STATUS.get(st, st), "rho": rep.rho, "x": x, "residual": rep.resid,
           "cycles": rep.cycles, "a_matvecs": rep.a_matvecs, "b_matvecs": rep.b_matvecs,
           "log": {k_: v[:L].copy() for k_, v in logs.items()}}
    if qopt_cap > 0:
        Lq = min(L, qopt_cap)
        out["log"]["qopt"] = qo[:Lq].copy()
        out["log"]["qdim"] = qd[:Lq].copy()
        if gl is not None:
            out["g"] = gl[:max(Lq - 1, 0)].T.copy()
    return out
