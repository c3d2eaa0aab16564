"""Measure kernel (a) gather_update (and (d) centroid) alone at full config
sizes: Eq.(3) sweeps with a trivial representative map (k = 1, parent =
identity) so that the repulsion part is negligible; reports the gather's
algorithmic bytes per launch / its CUDA-event time against the measured HBM
peak.  Usage: python tools/bench_gather.py cfg5 [cfg4 ...]"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1506_04383_b200 as mm  # noqa: E402
from workloads import configs  # noqa: E402

HBM = json.load(open(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json")))["hbm_gbs"] \
    if os.path.exists(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json")) else 6554.6

out = {}
for name in sys.argv[1:] or ["cfg5"]:
    w = configs.make(name)
    n, dim = w.n, w.dim
    S = mm.sset_to_device(w.S)
    x = mm.coords_to_device(configs.random_state(n, dim, seed=1, scale=n ** (1 / dim)))
    y = torch.empty_like(x)
    par = torch.arange(n, dtype=torch.int32, device="cuda")
    anc = torch.zeros(n, dtype=torch.int32, device="cuda")
    for _ in range(2):
        mm.sweep(S, x, w.alpha, w.q, parent=par, ancestor=anc, k=1, out=y)
    torch.cuda.synchronize()
    mm.profile_reset()
    mm.profile_enable(True)
    reps = 5
    for _ in range(reps):
        mm.sweep(S, x, w.alpha, w.q, parent=par, ancestor=anc, k=1, out=y)
    torch.cuda.synchronize()
    prof = mm.profile_read()
    mm.profile_enable(False)
    bx = 8 if dim == 2 else 16
    nnz = w.S.nnz
    # algorithmic bytes: S CSR once, x once, one partial slot, x_out once, parent + child CSR
    alg = 8 * (n + 1) + 12 * nnz + bx * n + bx * n + bx * n + 4 * n + 4 * (n + 1) + 4 * n
    g = prof["gather_update"]
    ms = g["total_ms"] / g["launches"]
    out[name] = {"n": n, "nnz": nnz, "gather_ms": ms, "alg_bytes": alg, "GBps": alg / (ms * 1e-3) / 1e9,
                 "hbm_frac": alg / (ms * 1e-3) / 1e9 / HBM, "G": os.environ.get("MM_GATHER_G", "auto")}
    print(name, json.dumps(out[name]), flush=True)
    del S, x, y
    torch.cuda.empty_cache()
