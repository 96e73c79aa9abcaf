"""Seeded synthetic inputs for BASELINE.json configs C1-C5 (and small variants).

Shared by the oracle tests and the CUDA path; holds none of TRPL+K's arithmetic
(DESIGN.md "Input recipe").  Matrices are CSR with int64 row pointers and
column ids, fp64 values, both triangles stored, columns strictly increasing
within a row (the shape SPEC.md S:22-28 gives for SparseSymMatrix).

The five configurations are the BASELINE.json ``configs`` list; the paper's
own matrices (Table 5.1) are not available and these
synthetic stencils stand in for them.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "gen.c")
_LIB = os.path.join(_HERE, "libgen.so")

SEED = 12  # PAPER.md:509 "fixed seed number(12)"


def build(force: bool = False) -> str:
    """Compile gen.c into libgen.so (plain gcc + OpenMP)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-o", _LIB, _SRC])
    return _LIB


_lib = None


def _get():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        lib.gen_u01.restype = ctypes.c_double
        lib.gen_u01.argtypes = [ctypes.c_uint64] * 3
        lib.gen_u01_fill.restype = None
        lib.gen_u01_fill.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64,
                                     ctypes.c_int64, ctypes.c_void_p]
        lib.gen_stencil_rowptr.restype = ctypes.c_int64
        lib.gen_stencil_rowptr.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int64,
                                           ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p]
        lib.gen_stencil_fill.restype = None
        lib.gen_stencil_fill.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int64,
                                         ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p,
                                         ctypes.c_void_p, ctypes.c_void_p, ctypes.c_double,
                                         ctypes.c_double, ctypes.c_double, ctypes.c_uint64]
        _lib = lib
    return _lib


def u01(seed: int, stream: int, index0: int, count: int) -> np.ndarray:
    """Counter-based U[0,1) draws (reading R13); index0.. index0+count-1."""
    out = np.empty(count, dtype=np.float64)
    _get().gen_u01_fill(seed, stream, index0, count, out.ctypes.data)
    return out


@dataclass
class CSR:
    n: int                 # global order
    row_begin: int         # first global row held
    rowptr: np.ndarray     # int64 [rows+1], local offsets
    col: np.ndarray        # int64 [nnz], global column ids
    val: np.ndarray        # float64 [nnz]

    @property
    def rows(self) -> int:
        return len(self.rowptr) - 1

    @property
    def nnz(self) -> int:
        return int(self.rowptr[-1])

    def to_scipy(self):
        import scipy.sparse as sp
        return sp.csr_matrix((self.val, self.col, self.rowptr), shape=(self.rows, self.n))


def stencil(dim: int, npts: int, N: int, center: float, off: float, dscale: float = 0.0,
            seed: int = SEED, row_begin: int = 0, row_end: Optional[int] = None) -> CSR:
    """dim=1: tridiag(off, center, off) of order N; dim=3: 7- or 27-point stencil on N^3.

    Diagonal = center + dscale*U(seed, stream 1, row) (reading R14)."""
    n = N if dim == 1 else N ** 3
    if row_end is None:
        row_end = n
    lib = _get()
    rows = row_end - row_begin
    rowptr = np.empty(rows + 1, dtype=np.int64)
    nnz = lib.gen_stencil_rowptr(dim, npts, N, row_begin, row_end, rowptr.ctypes.data)
    col = np.empty(nnz, dtype=np.int64)
    val = np.empty(nnz, dtype=np.float64)
    lib.gen_stencil_fill(dim, npts, N, row_begin, row_end, rowptr.ctypes.data, col.ctypes.data,
                         val.ctypes.data, float(center), float(off), float(dscale), seed)
    return CSR(n=n, row_begin=row_begin, rowptr=rowptr, col=col, val=val)


@dataclass
class Problem:
    name: str
    A: CSR
    B: Optional[CSR]
    p: int
    q: int          # max basis
    l: int          # k_plus
    tol: float
    sigma: float = 0.0
    desc: str = ""
    grid: dict = field(default_factory=dict)


# name -> (dim, N, A(npts, center, off, dscale), B(npts, center, off) | None, p, q, l, tol, desc)
CONFIGS = {
    "C1": (1, 1000, (3, 2.0, -1.0, 0.0), None, 5, 20, 1, 1e-8,
           "1D Dirichlet Laplacian tridiag(-1,2,-1), n=1000"),
    "C2": (3, 64, (7, 6.0, -1.0, 10.0), None, 10, 30, 2, 1e-8,
           "3D 7-pt Laplacian 64^3 + diag(d), d~U[0,10)"),
    "C3": (3, 128, (7, 6.0, -1.0, 0.0), None, 20, 48, 3, 1e-8,
           "3D 7-pt Laplacian 128^3 (clustered)"),
    "C4": (3, 160, (27, 26.0, -1.0, 1.0), (7, 1.0, 1.0 / 12.0), 10, 32, 2, 1e-8,
           "pencil 160^3: A 27-pt (26,-1)+diag(d), d~U[0,1); B 7-pt (1, 1/12)"),
    "C5": (3, 512, (7, 6.0, -1.0, 10.0), None, 8, 24, 2, 1e-7,
           "3D 7-pt Laplacian 512^3 + diag(d), d~U[0,10)"),
}


def make(name: str, N: Optional[int] = None, row_begin: int = 0, row_end: Optional[int] = None,
         seed: int = SEED, **over) -> Problem:
    """Build config `name` (C1..C5).  `N` overrides the grid size (tiny variants,
    e.g. make('C2', N=8)); `row_begin/row_end` restrict to a row slab (multi-GPU);
    keyword overrides replace p/q/l/tol/dscale (e.g. dscale=0 -> the d=0 variants)."""
    dim, N0, (npts, center, off, dscale), bspec, p, q, l, tol, desc = CONFIGS[name]
    N = N0 if N is None else N
    dscale = over.pop("dscale", dscale)
    A = stencil(dim, npts, N, center, off, dscale, seed, row_begin, row_end)
    B = None
    if bspec is not None:
        bn, bc, bo = bspec
        B = stencil(dim, bn, N, bc, bo, 0.0, seed, row_begin, row_end)
    prob = Problem(name=name, A=A, B=B, p=p, q=q, l=l, tol=tol, desc=desc,
                   grid={"dim": dim, "N": N, "npts": npts})
    for k, v in over.items():
        setattr(prob, k, v)
    return prob


def slab_rows(n: int, nranks: int, rank: int, plane: int = 1) -> tuple:
    """Contiguous row partition [r*n/P, (r+1)*n/P) rounded to whole planes."""
    planes = n // plane
    b = (planes * rank) // nranks
    e = (planes * (rank + 1)) // nranks
    return b * plane, (e * plane if rank < nranks - 1 else n)


def sample_rows(n: int, count: int = 2048, seed: int = SEED) -> np.ndarray:
    """Sorted distinct rows floor(U(seed, stream 8, i) * n), i < count: where full-size parity
    tests compare eigenvector entries with the oracle's (tests/golden/oracle_<cfg>.json)."""
    r = np.floor(u01(seed, 8, 0, count) * n).astype(np.int64)
    return np.unique(np.clip(r, 0, n - 1))
