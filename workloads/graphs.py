"""Seeded synthetic graph generators for the five BASELINE.json configs.

These stand in for the paper's instance classes (§4 "Instances",
P:339-350: FE meshes, Delaunay graphs of random points in the unit square,
road networks; largest connected component, unit edge lengths).  The paper's
files are not available; every graph here is synthetic and seeded.

This module is shared by the oracle tests, the GPU tests and bench.py.  It
holds NONE of the method's arithmetic (no Eq.(2)/(3), no matching, no
contraction): it only produces CSR graphs.

All graphs are returned as ``Graph(row_ptr int64[n+1], col int32[2m])``,
symmetric, no self loops, no duplicate edges, each row sorted ascending.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp
from scipy.sparse.csgraph import connected_components


@dataclass
class Graph:
    row_ptr: np.ndarray  # int64 [n+1]
    col: np.ndarray      # int32 [nnz]

    @property
    def n(self) -> int:
        return int(self.row_ptr.shape[0] - 1)

    @property
    def nnz(self) -> int:
        return int(self.col.shape[0])

    @property
    def m(self) -> int:
        return self.nnz // 2

    def degrees(self) -> np.ndarray:
        return np.diff(self.row_ptr)

    def to_scipy(self) -> sp.csr_matrix:
        data = np.ones(self.nnz, dtype=np.int8)
        return sp.csr_matrix((data, self.col, self.row_ptr), shape=(self.n, self.n))


def from_edges(n: int, u: np.ndarray, v: np.ndarray) -> Graph:
    """Undirected edge list -> symmetric CSR (dedup, no self loops, sorted rows)."""
    u = np.asarray(u, dtype=np.int64)
    v = np.asarray(v, dtype=np.int64)
    keep = u != v
    u, v = u[keep], v[keep]
    a = np.concatenate([u, v])
    b = np.concatenate([v, u])
    key = np.sort(a * n + b)
    if key.shape[0]:
        key = key[np.concatenate([[True], key[1:] != key[:-1]])]
    rows = (key // n).astype(np.int64)
    cols = (key % n).astype(np.int32)
    row_ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(rows, minlength=n), out=row_ptr[1:])
    return Graph(row_ptr, cols)


def largest_component(g: Graph) -> tuple[Graph, np.ndarray]:
    """Keep the LCC, relabelled preserving the original id order.

    Returns (graph, kept_ids) where kept_ids[new] = old."""
    ncomp, labels = connected_components(g.to_scipy(), directed=False)
    if ncomp == 1:
        return g, np.arange(g.n, dtype=np.int64)
    sizes = np.bincount(labels)
    big = int(np.argmax(sizes))
    kept = np.nonzero(labels == big)[0].astype(np.int64)
    newid = -np.ones(g.n, dtype=np.int64)
    newid[kept] = np.arange(kept.shape[0])
    rows = np.repeat(np.arange(g.n, dtype=np.int64), g.degrees())
    cols = g.col.astype(np.int64)
    mask = (newid[rows] >= 0) & (newid[cols] >= 0)
    nr, nc = newid[rows[mask]], newid[cols[mask]]
    n2 = kept.shape[0]
    row_ptr = np.zeros(n2 + 1, dtype=np.int64)
    np.cumsum(np.bincount(nr, minlength=n2), out=row_ptr[1:])
    # rows stay sorted: old order is preserved by the relabelling and the CSR
    # was already row-major sorted
    return Graph(row_ptr, nc.astype(np.int32)), kept


# ---------------------------------------------------------------- generators

def grid2d(rows: int, cols: int) -> Graph:
    """rows x cols grid, id = r*cols + c (configs[0]: 32x32)."""
    ids = np.arange(rows * cols, dtype=np.int64).reshape(rows, cols)
    u = np.concatenate([ids[:, :-1].ravel(), ids[:-1, :].ravel()])
    v = np.concatenate([ids[:, 1:].ravel(), ids[1:, :].ravel()])
    return from_edges(rows * cols, u, v)


def grid3d(a: int, b: int, c: int) -> Graph:
    """a x b x c grid, id = (i*b + j)*c + k (configs[4]: 128^3)."""
    ids = np.arange(a * b * c, dtype=np.int64).reshape(a, b, c)
    u = np.concatenate([ids[:-1].ravel(), ids[:, :-1].ravel(), ids[:, :, :-1].ravel()])
    v = np.concatenate([ids[1:].ravel(), ids[:, 1:].ravel(), ids[:, :, 1:].ravel()])
    return from_edges(a * b * c, u, v)


def trimesh(side: int, seed: int) -> Graph:
    """side x side grid plus one seeded diagonal per cell (configs[2]: 512)."""
    rng = np.random.default_rng(seed)
    ids = np.arange(side * side, dtype=np.int64).reshape(side, side)
    coin = rng.integers(0, 2, size=(side - 1, side - 1)).astype(bool)
    d1u, d1v = ids[:-1, :-1], ids[1:, 1:]      # (r,c)-(r+1,c+1)
    d2u, d2v = ids[:-1, 1:], ids[1:, :-1]      # (r,c+1)-(r+1,c)
    du = np.where(coin, d1u, d2u).ravel()
    dv = np.where(coin, d1v, d2v).ravel()
    u = np.concatenate([ids[:, :-1].ravel(), ids[:-1, :].ravel(), du])
    v = np.concatenate([ids[:, 1:].ravel(), ids[1:, :].ravel(), dv])
    return from_edges(side * side, u, v)


def rgg(n: int, seed: int, mean_degree: float = 8.0) -> tuple[Graph, np.ndarray]:
    """Random geometric graph in the unit square, radius for the given mean
    degree, LCC kept (configs[1]).  Stands in for the paper's Delaunay graphs
    del16/del20.  Returns (graph, points of the kept vertices)."""
    from scipy.spatial import cKDTree

    rng = np.random.default_rng(seed)
    pts = rng.random((n, 2))
    r = float(np.sqrt(mean_degree / (np.pi * n)))
    pairs = cKDTree(pts).query_pairs(r, output_type="ndarray")
    g = from_edges(n, pairs[:, 0], pairs[:, 1])
    g, kept = largest_component(g)
    return g, pts[kept]


def chung_lu_weights(n: int, mean: float = 10.0, wmax: float = 2000.0,
                     exponent: float = 2.5) -> np.ndarray:
    """Expected-degree sequence w_i = c (i + i0)^(-1/(exponent-1)), descending,
    with mean `mean` and w_0 = wmax (configs[3])."""
    gam = 1.0 / (exponent - 1.0)
    i = np.arange(n, dtype=np.float64)

    def mean_for(i0: float) -> float:
        c = wmax * i0 ** gam
        return float(np.mean(c * (i + i0) ** (-gam)))

    lo, hi = 1e-3, 1e7  # mean_for is increasing in i0: bisect on a log scale
    for _ in range(80):
        mid = np.sqrt(lo * hi)
        if mean_for(mid) < mean:
            lo = mid
        else:
            hi = mid
    i0 = np.sqrt(lo * hi)
    c = wmax * i0 ** gam
    return c * (i + i0) ** (-gam)


def chung_lu(n: int, seed: int, mean: float = 10.0, wmax: float = 2000.0,
             exponent: float = 2.5) -> Graph:
    """Chung-Lu power-law graph via Norros-Reittu-style sampling: Poisson(W/2)
    endpoint pairs drawn independently proportional to the expected degrees,
    self loops and multi-edges dropped; LCC kept.  Ids are in weight-descending
    order (id 0 = the heaviest vertex)."""
    rng = np.random.default_rng(seed)
    w = chung_lu_weights(n, mean, wmax, exponent)
    W = float(w.sum())
    m = int(rng.poisson(W / 2.0))
    cdf = np.cumsum(w) / W
    # sorted uniforms make the binary searches cache friendly; v is permuted
    # afterwards so that the two endpoints stay independent
    u = np.searchsorted(cdf, np.sort(rng.random(m)), side="right")
    v = rng.permutation(np.searchsorted(cdf, np.sort(rng.random(m)), side="right"))
    u = np.minimum(u, n - 1)
    v = np.minimum(v, n - 1)
    g = from_edges(n, u, v)
    g, _ = largest_component(g)
    return g
