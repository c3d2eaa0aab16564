"""Level-0 launches of the hierarchy kernels (d) and the prolongation, against
algorithmic bytes (builder tool; SURVEY §8(d) row "(d) match/contract/prolong":
HBM, ~12-16 B per directed edge per round, sort ~16 B nnz per pass).

torch.profiler (CUPTI) records every launch in order: the hierarchy is built
from level 0 upwards, so each kernel's FIRST launch is level 0's; the
layout prolongs to level 0 last, so k_prolong's LAST launch is level 0's.
Algorithmic bytes per launch (n = level-0 vertices, m = directed edges):
  k_match_level  rounds x (8 n row bounds + 8 m (col, omega) + 8 m (c, mate
                 of the neighbour) + 8 n (c, mate of the vertex) + 4 n cand)
  k_edge_keys    m x (4 row id + 4 col + 4 omega + 4 parent[col] + 8 key + 4 val)
  k_rs_scatter   m x (12 read + 12 write)      (one digit pass of sort_edges)
  k_rs_hist      m x 8                          (one digit pass)
  k_prolong      n x (4 parent + b_x parent coordinates + b_x out)
Usage: python tools/hier_kernels.py cfg5 cfg4"""
import json
import os
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1506_04383_b200 as mm  # noqa: E402
from workloads import configs  # noqa: E402

HBM = 6539.2


def main(name):
    w = configs.make(name)
    g = mm.graph_to_device(w.graph)
    S = mm.sset_to_device(w.S)
    H = mm.build_hierarchy(g, w.dim, w.seed)
    rounds0 = int(H.level_host(0)["rounds"])
    n, m = w.n, int(w.graph.nnz)
    bx = 8 if w.dim == 2 else 16
    mm.layout(g, S, w.dim, w.alpha, w.q, w.h, [w.sweeps], w.seed)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        mm.layout(g, S, w.dim, w.alpha, w.q, w.h, [w.sweeps], w.seed)
        torch.cuda.synchronize()
    evs = sorted([e for e in prof.events() if e.device_type.name == "CUDA"], key=lambda e: e.time_range.start)
    algo = {
        "k_match_level": ("first", rounds0 * (8 * n + 8 * m + 8 * m + 8 * n + 4 * n)),
        "k_edge_keys": ("first", m * 28),
        "k_rs_hist": ("first", m * 8),
        "k_rs_scatter": ("first", m * 24),
        "k_prolong": ("last", n * (4 + 2 * bx)),
    }
    out = {"config": name, "n": n, "m": m, "match_rounds_level0": rounds0}
    for kern, (which, by) in algo.items():
        ts = [e.time_range.elapsed_us() for e in evs if kern in e.name and "disc" not in e.name]
        if not ts:
            continue
        us = ts[0] if which == "first" else ts[-1]
        gbs = by / (us * 1e-6) / 1e9
        out[kern] = {"us": us, "algo_bytes": by, "GBps": gbs, "frac_hbm": gbs / HBM}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    for nm in sys.argv[1:]:
        main(nm)
