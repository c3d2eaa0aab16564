"""Full-size check of mm_energy (kernel (e)) on the largest config (builder tool).

Step 1 (GPU):  python tests/tools/energy_fullsize_check.py gpu cfg5 OUT.npz
    runs one mm_layout of the config and saves the final layout x (float32) with the energy terms
    mm_layout reported for it.
Step 2 (CPU):  python tests/tools/energy_fullsize_check.py oracle cfg5 OUT.npz
    evaluates the FP64 oracle's energy (oracle/ only: every unordered pair, about 2.2e12 pow calls at
    cfg5) of that layout and prints both with their relative differences.
The oracle's own full run of cfg5 is infeasible (~7.5 days single-threaded); this pins
the energy kernel, not the run, at full size."""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from workloads import configs  # noqa: E402


def gpu(name, out):
    import torch

    import paper_1506_04383_b200 as mm

    w = configs.make(name)
    x, rep = mm.layout(mm.graph_to_device(w.graph), mm.sset_to_device(w.S), w.dim, w.alpha, w.q, w.h, [w.sweeps],
                       w.seed)
    torch.cuda.synchronize()
    np.savez(out, x=mm.coords_from_device(x, w.dim).astype(np.float32),
             terms=np.asarray([rep["stress"], rep["entropy"], rep["energy"]], dtype=np.float64),
             coincident=np.asarray([rep["coincident_pairs"]]))
    print(json.dumps({"config": name, "stress": rep["stress"], "entropy": rep["entropy"], "energy": rep["energy"]}))


def cpu(name, out):
    import oracle

    w = configs.make(name)
    z = np.load(out)
    x = z["x"].astype(np.float64)
    t = time.perf_counter()
    eo = oracle.energy(w.S, x, w.alpha, w.q)
    secs = time.perf_counter() - t
    tg = z["terms"]
    rel = [abs(tg[i] - eo[i]) / max(abs(eo[i]), 1e-300) for i in range(3)]
    print(json.dumps({"config": name, "n": int(w.n), "gpu": {"stress": tg[0], "entropy": tg[1], "energy": tg[2]},
                      "oracle": {"stress": eo[0], "entropy": eo[1], "energy": eo[2]},
                      "rel": {"stress": rel[0], "entropy": rel[1], "energy": rel[2]},
                      "oracle_seconds": secs, "oracle_threads": oracle.default_threads()}), flush=True)


if __name__ == "__main__":
    {"gpu": gpu, "oracle": cpu}[sys.argv[1]](sys.argv[2], sys.argv[3])
