"""Small hand-made instances for the oracle pins (no method arithmetic)."""
from __future__ import annotations

import os

import numpy as np

from workloads import graphs, sset

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def read_golden(name: str) -> np.ndarray:
    rows = []
    with open(os.path.join(GOLDEN, name)) as f:
        for line in f:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            rows.append([float(t) for t in line.split()])
    return np.array(rows, dtype=np.float64)


def path(n: int) -> graphs.Graph:
    return graphs.from_edges(n, np.arange(n - 1), np.arange(1, n))


def cycle(n: int) -> graphs.Graph:
    return graphs.from_edges(n, np.arange(n), (np.arange(n) + 1) % n)


def petersen() -> graphs.Graph:
    outer = [(i, (i + 1) % 5) for i in range(5)]
    spokes = [(i, i + 5) for i in range(5)]
    inner = [(5 + i, 5 + (i + 2) % 5) for i in range(5)]
    e = np.array(outer + spokes + inner)
    return graphs.from_edges(10, e[:, 0], e[:, 1])


def random_connected(n: int, extra: int, seed: int) -> graphs.Graph:
    """Random spanning tree plus `extra` random edges."""
    rng = np.random.default_rng(seed)
    par = np.array([rng.integers(0, i) for i in range(1, n)])
    u = np.concatenate([np.arange(1, n), rng.integers(0, n, extra)])
    v = np.concatenate([par, rng.integers(0, n, extra)])
    return graphs.from_edges(n, u, v)


def sset_with(g: graphs.Graph, d: np.ndarray) -> sset.SSet:
    """S = E with given per-entry d (must be symmetric), w = d^-2."""
    d = np.asarray(d, dtype=np.float64)
    return sset.SSet(g.row_ptr.copy(), g.col.copy(), d, 1.0 / (d * d))


def symmetric_random_d(g: graphs.Graph, lo: float, hi: float, seed: int) -> np.ndarray:
    """Random symmetric per-edge values on a CSR graph."""
    rng = np.random.default_rng(seed)
    n = g.n
    rows = np.repeat(np.arange(n), g.degrees())
    a = np.minimum(rows, g.col)
    b = np.maximum(rows, g.col)
    key = a.astype(np.int64) * n + b
    uk, inv = np.unique(key, return_inverse=True)
    vals = rng.uniform(lo, hi, uk.shape[0])
    return vals[inv]
