"""Kernel (b) exact repulsion: symmetric (MM_SYM=1, default) vs one-sided
(MM_SYM=0).  Run once per mode (the library reads MM_SYM once per process);
prints per-launch repulse_exact / gather_update times, pairs/s, and dumps the
layout after `reps` sweeps to /tmp for a cross-mode comparison.
Usage: MM_SYM=0|1 python tools/bench_sym.py cfg2 [cfg1_grid64 ...]"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1506_04383_b200 as mm  # noqa: E402
from workloads import configs  # noqa: E402

mode = os.environ.get("MM_SYM", "1")
for name in sys.argv[1:] or ["cfg2"]:
    w = configs.make(name)
    n, dim = w.n, w.dim
    S = mm.sset_to_device(w.S)
    x0 = mm.coords_to_device(configs.random_state(n, dim, seed=1, scale=n ** (1 / dim)))
    x = x0.clone()
    y = torch.empty_like(x)
    for _ in range(3):
        mm.sweep(S, x, w.alpha, w.q, out=y)
    torch.cuda.synchronize()
    mm.profile_reset()
    mm.profile_enable(True)
    reps = 10
    for _ in range(reps):
        mm.sweep(S, x, w.alpha, w.q, out=y)
    torch.cuda.synchronize()
    prof = mm.profile_read()
    mm.profile_enable(False)
    r = prof["repulse_exact"]
    ms = r["total_ms"] / r["launches"]
    pairs = n * (n - 1)
    res = {"mode": mode, "n": n, "repulse_ms": ms, "ordered_pairs_per_s": pairs / (ms * 1e-3),
           "gather_ms": prof["gather_update"]["total_ms"] / prof["gather_update"]["launches"]}
    print(name, json.dumps(res), flush=True)
    # iterate a few sweeps for the cross-mode comparison
    x = x0.clone()
    for _ in range(5):
        mm.sweep(S, x, w.alpha, w.q, out=y)
        x, y = y, x
    np.save(f"gpurun_out/sym_{name}_{mode}.npy", x.cpu().numpy())
