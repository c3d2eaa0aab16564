"""Full-run parity at FULL config size (Q20): the GPU mm_layout run
against the FP64 oracle's own full run of the same config, on the GPU box's
host cores (OpenMP over rows).  Prints one JSON line per config:
E_gpu, E_oracle, their relative difference (bar 1e-3), the oracle energy of
the GPU layout (kernel error isolated from trajectory divergence) and times.
Usage: python tests/tools/fullrun_parity.py cfg2 cfg3"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import oracle  # noqa: E402
import paper_1506_04383_b200 as mm  # noqa: E402
from workloads import configs  # noqa: E402

for name in sys.argv[1:] or ["cfg2", "cfg3"]:
    w = configs.make(name)
    S = mm.sset_to_device(w.S)
    g = mm.graph_to_device(w.graph) if w.h > 0 else None
    x0 = mm.coords_to_device(w.x0) if w.h == 0 else None
    t = time.perf_counter()
    x, rep = mm.layout(g, S, w.dim, w.alpha, w.q, w.h, [w.sweeps], w.seed, x_init=x0)
    torch.cuda.synchronize()
    t_gpu = time.perf_counter() - t
    xg = mm.coords_from_device(x, w.dim)
    t = time.perf_counter()
    xo, eo, nl = oracle.layout(w.graph, w.S, w.dim, w.alpha, w.q, w.h, [w.sweeps], w.seed,
                               x_init=None if w.h > 0 else w.x0.astype(np.float64))
    t_or = time.perf_counter() - t
    rel = abs(rep["energy"] - eo[2]) / abs(eo[2])
    res = {"config": name, "n": w.n, "levels_gpu": rep["levels"], "levels_oracle": nl,
           "E_gpu": rep["energy"], "E_oracle": eo[2], "rel_diff": rel, "within_1e-3": rel <= 1e-3,
           "stress_gpu": rep["stress"], "stress_oracle": eo[0], "coincident_pairs_gpu": rep["coincident_pairs"],
           "gpu_s": t_gpu, "oracle_s": t_or, "oracle_threads": oracle.default_threads()}
    print(json.dumps(res), flush=True)
    # kernel error alone: the oracle's energy of the GPU layout; FP32 layouts can hold exactly
    # coincident vertices (leaves of one hub), left out as the GPU report does (Q6)
    eg = oracle.energy(w.S, xg.astype(np.float64), w.alpha, w.q, skip_coincident=True)
    res.update({"E_oracle_of_gpu_layout": eg[2], "rel_kernel": abs(rep["energy"] - eg[2]) / abs(eg[2])})
    print(json.dumps(res), flush=True)
