"""Fraction of (warp, source tile) pairs of kernel (c) that take the lo-free far
path (Q27) on the final finest-level layout of a config, for several
thresholds 2^-b X.  Orders, frame origin (Q28) and boxes are recomputed here on
the host (numpy) the way approx_orders / k_frame / k_tile_box define them.
Usage: python tools/far_fraction.py cfg4 [cfg3 ...]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1506_04383_b200 as mm  # noqa: E402
from workloads import configs  # noqa: E402


def morton(p, lo, hi, bits):
    ext = np.where(hi > lo, hi - lo, 1.0)
    q = np.clip(((p - lo) / ext * (1 << bits)).astype(np.int64), 0, (1 << bits) - 1)
    key = np.zeros(len(p), np.int64)
    for b in range(bits):
        for c in range(p.shape[1]):
            key |= ((q[:, c] >> b) & 1) << (b * p.shape[1] + c)
    return key


for name in sys.argv[1:] or ["cfg4"]:
    w = configs.make(name)
    g = mm.graph_to_device(w.graph)
    S = mm.sset_to_device(w.S)
    x, rep = mm.layout(g, S, w.dim, w.alpha, w.q, w.h, [w.sweeps], w.seed)
    torch.cuda.synchronize()
    X = mm.coords_from_device(x, w.dim).astype(np.float64)
    H = mm.build_hierarchy(g, w.dim, w.seed)
    p0 = H.level_host(0)["parent"]
    p1 = H.level_host(1)["parent"]
    anc = p1[p0]
    k = int(anc.max()) + 1
    n, dim = X.shape
    nu = np.bincount(anc, minlength=k)
    cen = np.stack([np.bincount(anc, weights=X[:, c], minlength=k) for c in range(dim)], 1) / nu[:, None]
    lo, hi = X.min(0), X.max(0)
    bits = 16 if dim == 2 else 10
    tord = np.argsort(morton(X, lo, hi, bits), kind="stable")
    rkey = (nu.astype(np.int64) << 32) | morton(cen, lo, hi, bits)
    # frame origin (Q28): box midpoint where it keeps x - c exact, else 0
    m = 0.5 * lo + 0.5 * hi
    c = np.where(((lo > 0) & (0.5 * m <= lo) & (hi <= 2 * m)) | ((hi < 0) & (0.5 * m >= hi) & (lo >= 2 * m)), m, 0.0)
    X = X - c
    cen = cen - c
    rord = np.argsort(rkey, kind="stable")
    T = 128 if dim == 2 else 64
    nw = (n + T - 1) // T
    tp = np.concatenate([tord, np.full(nw * T - n, tord[-1])])
    tx = X[tp].reshape(nw, T, dim)
    wlo, whi = tx.min(1), tx.max(1)
    wX = np.maximum(np.abs(wlo), np.abs(whi)).max(1)
    nt = (k + 255) // 256
    rp = np.concatenate([rord, np.full(nt * 256 - k, rord[-1])])
    rc = cen[rp].reshape(nt, 256, dim)
    blo, bhi = rc.min(1), rc.max(1)
    bX = np.maximum(np.abs(blo), np.abs(bhi)).max(1)
    res = {}
    for b in (7, 9, 11):
        far = 0
        for i0 in range(0, nw, 512):
            sl = slice(i0, i0 + 512)
            sep = np.maximum(0, np.maximum(blo[None] - whi[sl, None], wlo[sl, None] - bhi[None]))
            d2 = (sep ** 2).sum(-1)
            XX = np.maximum(wX[sl, None], bX[None])
            far += int((d2 >= (XX * 2.0 ** -b) ** 2).sum())
        res[b] = far / (nw * nt)
    wext = (whi - wlo).max(1)
    bext = (bhi - blo).max(1)
    print(name, f"n={n} k={k} X={np.abs(X).max():.4g} extent={(hi - lo).max():.4g}",
          f"warp box median {np.median(wext):.3g} tile box median {np.median(bext):.3g}",
          "far fraction by 2^-b:", res, flush=True)
