"""Wall time of mm_layout_schedule vs the sum of its kernels' device time
(library CUDA events): the difference is host round trips and launch gaps.
Usage: python tools/sched_overhead.py cfg2 7"""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1506_04383_b200 as mm  # noqa: E402
from workloads import configs  # noqa: E402

name, h = sys.argv[1], int(sys.argv[2])
w = configs.make(name)
G, S = mm.graph_to_device(w.graph), mm.sset_to_device(w.S)
sch = mm.paper_schedule(max_final_iters=200)
for sc in (False, True):
    mm.layout_schedule(G, S, w.dim, w.q, h, sch, w.seed, sclap=sc, disc=sc)
    torch.cuda.synchronize()
    t = time.perf_counter()
    x, rep = mm.layout_schedule(G, S, w.dim, w.q, h, sch, w.seed, sclap=sc, disc=sc)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t
    mm.profile_reset()
    mm.profile_enable(True)
    mm.layout_schedule(G, S, w.dim, w.q, h, sch, w.seed, sclap=sc, disc=sc)
    torch.cuda.synchronize()
    prof = mm.profile_read()
    mm.profile_enable(False)
    dev = sum(v["total_ms"] for v in prof.values())
    launches = sum(v["launches"] for v in prof.values())
    print(json.dumps({"config": name, "h": h, "sclap": sc, "wall_ms": wall * 1e3, "kernel_ms": dev,
                      "launches": launches, "sweeps": sum(rep["sweeps_level"]),
                      "top": {k: round(v["total_ms"], 2) for k, v in sorted(prof.items(), key=lambda kv: -kv[1]["total_ms"])[:6]}}))
