"""Kernel (d) centroid at full config sizes: one Eq.(3) sweep per call with the
finest level's map to level h (h = 2: the BASELINE configs, h = 7: MulMent_7),
per-launch CUDA-event time, algorithmic bytes (member ids 4 B + member coords
b_x per member, mptr 4 B + hi/lo 32 B per representative) against the measured
HBM peak.  Usage: python tools/bench_centroid.py cfg5 cfg4 cfg3"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1506_04383_b200 as mm  # noqa: E402
from workloads import configs  # noqa: E402

HBM = 6554.6
for name in sys.argv[1:] or ["cfg5"]:
    w = configs.make(name)
    n, dim = w.n, w.dim
    H = mm.build_hierarchy(mm.graph_to_device(w.graph), dim, w.seed)
    lv = [H.level_host(l) for l in range(H.num_levels)]
    S = mm.sset_to_device(w.S)
    x = mm.coords_to_device(configs.random_state(n, dim, seed=1, scale=n ** (1 / dim)))
    y = torch.empty_like(x)
    for h in (2, 7):
        if h >= len(lv):
            continue
        anc = np.arange(n)
        for l in range(h):
            anc = lv[l]["parent"][anc]
        k = lv[h]["n"]
        par = torch.from_numpy(lv[0]["parent"].astype(np.int32)).cuda()
        ancd = torch.from_numpy(anc.astype(np.int32)).cuda()
        mm.sweep(S, x, w.alpha, w.q, parent=par, ancestor=ancd, k=k, out=y)
        torch.cuda.synchronize()
        mm.profile_reset()
        mm.profile_enable(True)
        for _ in range(3):
            mm.sweep(S, x, w.alpha, w.q, parent=par, ancestor=ancd, k=k, out=y)
        torch.cuda.synchronize()
        prof = mm.profile_read()
        mm.profile_enable(False)
        c = prof["centroid"]
        ms = c["total_ms"] / c["launches"]
        bx = 8 if dim == 2 else 16
        alg = (4 + bx) * n + 36 * k
        print(name, json.dumps({"h": h, "n": n, "k": k, "centroid_ms": ms, "GBps": alg / (ms * 1e-3) / 1e9,
                                "hbm_frac": alg / (ms * 1e-3) / 1e9 / HBM}), flush=True)
