"""Stress pair sets S (inputs of the method; PAPER.md P:163 footnote: "the
stress term for arbitrary supersets S ⊇ E"; w = d^-2).

Each builder returns ``SSet(row_ptr int64[n+1], col int32[nnz], d float64[nnz],
w float64[nnz])``: per-vertex rows S_i, sorted ascending within the row
except for the capped builder (edges first, then hop-2 vertices, both
ascending).  d is the hop distance, w = d^-2, exactly as BASELINE.json's
configs state; these are input definitions, not method arithmetic.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp

from .graphs import Graph

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = os.path.join(_HERE, "libmmgen.so")


@dataclass
class SSet:
    row_ptr: np.ndarray  # int64 [n+1]
    col: np.ndarray      # int32 [nnz]
    d: np.ndarray        # float64 [nnz]
    w: np.ndarray        # float64 [nnz]

    @property
    def n(self) -> int:
        return int(self.row_ptr.shape[0] - 1)

    @property
    def nnz(self) -> int:
        return int(self.col.shape[0])

    def row_lengths(self) -> np.ndarray:
        return np.diff(self.row_ptr)


def edges_sset(g: Graph, d: float = 1.0) -> SSet:
    """S = E, d_ij = d, w_ij = d^-2 (configs[0], configs[4])."""
    dd = np.full(g.nnz, d, dtype=np.float64)
    return SSet(g.row_ptr.copy(), g.col.copy(), dd, 1.0 / (dd * dd))


def hop2_sset(g: Graph) -> SSet:
    """S_i = {j != i : hop(i,j) <= 2}, d = hop distance, w = d^-2
    (configs[1], configs[2])."""
    a = g.to_scipy().astype(np.int64)
    a2 = (a @ a).tocsr()
    big = np.int64(1) << 40
    s = (a * big + a2).tocsr()  # entries >= big are edges (hop 1)
    s.setdiag(0)
    s.eliminate_zeros()
    s.sort_indices()
    d = np.where(s.data >= big, 1.0, 2.0)
    return SSet(s.indptr.astype(np.int64), s.indices.astype(np.int32), d, 1.0 / (d * d))


def _lib() -> ctypes.CDLL:
    src = os.path.join(_HERE, "csrc", "capped2hop.c")
    if (not os.path.exists(_LIB)) or os.path.getmtime(_LIB) < os.path.getmtime(src):
        build()
    lib = ctypes.CDLL(_LIB)
    i64p = ctypes.POINTER(ctypes.c_int64)
    i32p = ctypes.POINTER(ctypes.c_int32)
    lib.gen_capped2hop.argtypes = [ctypes.c_int32, i64p, i32p, ctypes.c_int32, i32p, i32p]
    return lib


def build() -> None:
    src = os.path.join(_HERE, "csrc", "capped2hop.c")
    subprocess.check_call(["gcc", "-O2", "-shared", "-fPIC", "-o", _LIB, src])


def _p(a: np.ndarray, t):
    return a.ctypes.data_as(ctypes.POINTER(t))


def capped_sset(g: Graph, cap: int = 64) -> SSet:
    """S_i = N(i) ∪ {the `cap` lowest-id vertices at hop distance exactly 2}
    (configs[3]); rows hold the edges first, then the hop-2 ids, each part
    ascending.  Asymmetric in general (the cap is per row)."""
    lib = _lib()
    rp = np.ascontiguousarray(g.row_ptr, dtype=np.int64)
    col = np.ascontiguousarray(g.col, dtype=np.int32)
    out = np.empty((g.n, cap), dtype=np.int32)
    cnt = np.zeros(g.n, dtype=np.int32)
    if lib.gen_capped2hop(g.n, _p(rp, ctypes.c_int64), _p(col, ctypes.c_int32), cap,
                          _p(out, ctypes.c_int32), _p(cnt, ctypes.c_int32)) != 0:
        raise MemoryError("capped2hop failed")
    deg = g.degrees()
    rl = deg + cnt
    srp = np.zeros(g.n + 1, dtype=np.int64)
    np.cumsum(rl, out=srp[1:])
    nnz = int(srp[-1])
    scol = np.empty(nnz, dtype=np.int32)
    hop = np.empty(nnz, dtype=np.float64)
    # position of each edge entry: srp[row] + (k - rp[row])
    rows_e = np.repeat(np.arange(g.n, dtype=np.int64), deg)
    pos_e = srp[rows_e] + (np.arange(g.nnz, dtype=np.int64) - rp[rows_e])
    scol[pos_e] = col
    hop[pos_e] = 1.0
    # hop-2 entries follow the edges of each row
    mask = np.arange(cap, dtype=np.int32)[None, :] < cnt[:, None]
    rows_h = np.nonzero(mask)[0].astype(np.int64)
    slot = np.nonzero(mask)[1].astype(np.int64)
    pos_h = srp[rows_h] + deg[rows_h] + slot
    scol[pos_h] = out[mask]
    hop[pos_h] = 2.0
    return SSet(srp, scol, hop, 1.0 / (hop * hop))


def is_symmetric(s: SSet) -> bool:
    n = s.n
    m = sp.csr_matrix((s.d, s.col, s.row_ptr), shape=(n, n))
    diff = m - m.T
    return diff.nnz == 0 or np.abs(diff.data).max() == 0
