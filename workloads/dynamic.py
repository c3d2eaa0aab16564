"""Dynamic-graph perturbation model of PAPER.md §4.3, an input
generator for the dynamic update mode (no method arithmetic):

"we start with an input graph G and perform a breadth first search from a
random start node to compute a random spanning tree.  We then remove x%
undirected non-tree edges at random ...  Afterwards, we insert x% new edges
as follows.  We pick a random node and insert an undirected edge to a random
node that has distance 1 < d <= D in the original graph G."
"""
from __future__ import annotations

import numpy as np
from scipy.sparse.csgraph import breadth_first_order, dijkstra

from .graphs import Graph, from_edges


def perturb(g: Graph, x_percent: float, D: int, seed: int) -> Graph:
    rng = np.random.default_rng(seed)
    n = g.n
    A = g.to_scipy()
    start = int(rng.integers(0, n))
    _, pred = breadth_first_order(A, start, directed=False, return_predecessors=True)
    tree = set()
    for v in range(n):
        p = pred[v]
        if p >= 0:
            tree.add((min(v, p), max(v, p)))
    rows = np.repeat(np.arange(n), g.degrees())
    mask = rows < g.col
    eu, ev = rows[mask], g.col[mask].astype(np.int64)
    m = eu.shape[0]
    non_tree = np.array([i for i in range(m) if (int(eu[i]), int(ev[i])) not in tree], dtype=np.int64)
    k = int(round(m * x_percent / 100.0))
    drop = set(rng.choice(non_tree, size=min(k, non_tree.shape[0]), replace=False).tolist())
    keep = np.array([i for i in range(m) if i not in drop], dtype=np.int64)
    nu, nv = list(eu[keep]), list(ev[keep])
    added = 0
    tries = 0
    while added < k and tries < 100 * (k + 1):
        tries += 1
        u = int(rng.integers(0, n))
        dist = dijkstra(A, directed=False, indices=u, unweighted=True, limit=D)
        cand = np.nonzero((dist > 1) & (dist <= D))[0]
        if cand.shape[0] == 0:
            continue
        v = int(rng.choice(cand))
        nu.append(u)
        nv.append(v)
        added += 1
    return from_edges(n, np.array(nu), np.array(nv))
