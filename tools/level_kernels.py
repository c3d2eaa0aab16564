"""Per-launch kernel times of the FINEST level of an mm_layout run (builder
tool): torch.profiler (CUPTI) records every launch in order; the finest level
runs last, so its K sweeps are the last K launches of each per-sweep kernel.
Prints kernels (a) and (d) against SURVEY §8(d)'s algorithmic bytes:
  gather:   4 (n + 1) + 12 nnz + 3 b_x n
  centroid: (b_x + 4) n + b_x k
Usage: python tools/level_kernels.py cfg5 [cfg4 ...]   (MM_RENUMBER=0 for A/B)"""
import json
import os
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1506_04383_b200 as mm  # noqa: E402
from workloads import configs  # noqa: E402

HBM = 6539.2  # GB/s, MEASURED_PEAKS.json


def main(name):
    w = configs.make(name)
    g = mm.graph_to_device(w.graph)
    S = mm.sset_to_device(w.S)
    mm.layout(g, S, w.dim, w.alpha, w.q, w.h, [w.sweeps], w.seed)  # warm (graphs, pools)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        x, rep = mm.layout(g, S, w.dim, w.alpha, w.q, w.h, [w.sweeps], w.seed)
        torch.cuda.synchronize()
    evs = [e for e in prof.events() if e.device_type.name == "CUDA"]
    evs.sort(key=lambda e: e.time_range.start)
    K = w.sweeps
    k = rep["k_level"][0]
    bx = 8 if w.dim == 2 else 16
    algo = {"k_gather": 4 * (w.n + 1) + 12 * w.S.nnz + 3 * bx * w.n, "k_centroid": (bx + 4) * w.n + bx * k}
    out = {"config": name, "n": w.n, "k": k, "nnz": int(w.S.nnz), "renumber": os.environ.get("MM_RENUMBER", "1")}
    for kern in ("k_gather", "k_centroid", "k_repulse<", "k_tile_box", "k_frame_fused"):
        ts = [e.time_range.elapsed_us() for e in evs if kern in e.name]
        last = ts[-K:]
        if not last:
            continue
        us = sorted(last)[len(last) // 2]
        rec = {"median_us": us, "launches_level0": len(last)}
        if kern in algo:
            gbs = algo[kern] / (us * 1e-6) / 1e9
            rec.update({"algo_bytes": algo[kern], "GBps": gbs, "frac_hbm": gbs / HBM})
        out[kern.rstrip("<")] = rec
    # one-off per-level work of the finest level (renumbering, orders)
    for kern in ("k_permute_rows", "k_slot_fill", "k_permute_x", "k_scan_out", "k_rs_hist", "k_rs_scatter",
                 "DeviceRadixSort", "k_scan_sums"):
        ts = [e.time_range.elapsed_us() for e in evs if kern in e.name]
        if ts:
            out[kern] = {"total_us_all_levels": sum(ts), "launches": len(ts)}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    for nm in sys.argv[1:]:
        main(nm)
