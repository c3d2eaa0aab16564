"""Time mm_build_hierarchy per kernel (library CUDA events) at full config
sizes and report algorithmic bytes / time for the matching kernels.
Usage: python tools/bench_hier.py cfg5 cfg4 cfg3"""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1506_04383_b200 as mm  # noqa: E402
from workloads import configs  # noqa: E402

HBM = 6554.6
SCLAP = os.environ.get("SCLAP", "0") == "1"
for name in sys.argv[1:] or ["cfg5"]:
    w = configs.make(name)
    g = mm.graph_to_device(w.graph)
    H = mm.build_hierarchy(g, w.dim, w.seed, sclap=SCLAP)  # warm-up
    del H
    torch.cuda.synchronize()
    mm.profile_reset()
    mm.profile_enable(True)
    t0 = time.perf_counter()
    H = mm.build_hierarchy(g, w.dim, w.seed, sclap=SCLAP)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    prof = mm.profile_read()
    mm.profile_enable(False)
    levels = [H.view(l) for l in range(H.num_levels)]
    rounds = [v.rounds for v in levels]
    # algorithmic bytes of the matching rounds: per round and vertex 8 B row_ptr + 4 B mate + 4 B cand;
    # per directed edge 4 B col + 4 B omega + 4 B mate[v] + 4 B c[v]  (level sizes x rounds)
    mb = 0
    for l, v in enumerate(levels[:-1]):
        mb += rounds[l] * (16 * v.n + 16 * v.nnz)
    pick = prof.get("match_level", prof.get("match_pick", {"total_ms": float("nan")}))
    conf = prof.get("match_confirm", {"total_ms": float("nan")})
    tot_ms = sum(p["total_ms"] for p in prof.values())
    res = {"n": w.n, "levels": [v.n for v in levels], "rounds": rounds, "wall_ms": wall * 1e3,
           "kernel_ms": tot_ms, "match_ms (all rounds: match_level, or pick+confirm)": pick["total_ms"] + (0 if "match_level" in prof else conf["total_ms"]),
           "match_pick_ms": pick["total_ms"], "match_confirm_ms": conf["total_ms"],
           "match_pick_GBps": mb / (pick["total_ms"] * 1e-3) / 1e9,
           "match_pick_hbm_frac": mb / (pick["total_ms"] * 1e-3) / 1e9 / HBM,
           "kernels": {k: round(v["total_ms"], 3) for k, v in sorted(prof.items(), key=lambda kv: -kv[1]["total_ms"])}}
    print(("sclap " if SCLAP else "") + name, json.dumps(res), flush=True)
