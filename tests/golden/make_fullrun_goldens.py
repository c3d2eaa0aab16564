"""Writes tests/golden/fullrun_<config>.json: the FP64 oracle's own full
multilevel run (fixed alpha, the config's sweeps per level) of a
BASELINE.json config, and its final energy Eq.(1) (S form, Q3/Q4).

This script calls only `oracle/` and the seeded input generators in
`workloads/` (no CUDA path).  The -m gpu full-run tests
(tests/test_gpu_fullrun.py) compare mm_layout's final energy with these values
at the north_star bar (1e-3 relative).  The oracle's result does not depend on
its thread count (OpenMP over rows, each row summed in a fixed order).

Usage: python tests/golden/make_fullrun_goldens.py cfg2 cfg3 cfg4 cfg5_grid64
"""
from __future__ import annotations

import json
import os
import platform
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from workloads import configs  # noqa: E402


def golden_path(name: str) -> str:
    return os.path.join(ROOT, "tests", "golden", f"fullrun_{name}.json")


def run(name: str) -> dict:
    w = configs.make(name)
    t = time.perf_counter()
    x_init = None if w.h > 0 else w.x0.astype(np.float64)
    xo, eo, nl = oracle.layout(w.graph, w.S, w.dim, w.alpha, w.q, w.h, [w.sweeps], w.seed, x_init=x_init)
    secs = time.perf_counter() - t
    return {
        "config": name, "n": int(w.n), "nnz_S": int(w.S.nnz), "dim": w.dim, "alpha": w.alpha, "q": w.q,
        "h": w.h, "sweeps_per_level": w.sweeps, "seed": w.seed, "n_stop": 1000, "levels": int(nl),
        "stress": eo[0], "entropy": eo[1], "energy": eo[2],
        "bbox_diameter": float(np.linalg.norm(xo.max(axis=0) - xo.min(axis=0))),
        "oracle_seconds": secs, "oracle_threads": oracle.default_threads(),
        "host": platform.processor() or platform.machine(),
        "written_by": "tests/golden/make_fullrun_goldens.py (oracle/ only)",
        "cite": "energy Eq.(1) P:163-171; driver P:195-257; bar: BASELINE.json north_star 1e-3 relative",
    }


if __name__ == "__main__":
    for name in sys.argv[1:]:
        res = run(name)
        with open(golden_path(name), "w") as f:
            json.dump(res, f, indent=1)
            f.write("\n")
        print(json.dumps(res), flush=True)
