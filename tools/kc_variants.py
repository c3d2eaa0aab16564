"""Kernel (c) A/B harness: one finest-level Eq.(3) sweep of a multilevel
config on its final layout, timed per library build (builder tool, not a test).

  python tools/kc_variants.py build NAME -DMM_POLY_MASK3=0x25 ...   # here: builds tools/kc_libs/NAME.so
  python tools/kc_variants.py prepare cfg5                          # GPU: layout + maps -> /tmp/kc_cfg5.npz
  python tools/kc_variants.py time cfg5 tools/kc_libs/A.so ...      # GPU: one subprocess per library

Prints one JSON line per library: kernel (c) ms per launch (library CUDA
events, median of 3) and pairs/s = n (k - 1) / time."""
from __future__ import annotations

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
LIBS = os.path.join(ROOT, "tools", "kc_libs")


def prepare(name):
    import numpy as np
    import torch

    import paper_1506_04383_b200 as mm
    from workloads import configs

    w = configs.make(name)
    g = mm.graph_to_device(w.graph)
    S = mm.sset_to_device(w.S)
    x, rep = mm.layout(g, S, w.dim, w.alpha, w.q, w.h, [w.sweeps], w.seed)
    H = mm.build_hierarchy(g, w.dim, w.seed)
    p0 = H.level_host(0)["parent"]
    p1 = H.level_host(1)["parent"]
    anc = p1[p0].astype(np.int32)
    k = int(H.view(2).n)
    torch.cuda.synchronize()
    np.savez(f"/tmp/kc_{name}.npz", x=x.cpu().numpy(), p0=p0.astype(np.int32), anc=anc, k=k)


def time_one(name, lib):
    os.environ["MM_LIB_PATH"] = lib
    import numpy as np
    import torch

    import paper_1506_04383_b200 as mm
    from workloads import configs

    w = configs.make(name)
    z = np.load(f"/tmp/kc_{name}.npz")
    S = mm.sset_to_device(w.S)
    x = torch.from_numpy(z["x"]).cuda()
    par = torch.from_numpy(z["p0"]).cuda()
    anc = torch.from_numpy(z["anc"]).cuda()
    k = int(z["k"])
    mm.sweep(S, x, w.alpha, w.q, parent=par, ancestor=anc, k=k)
    torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        mm.profile_reset()
        mm.profile_enable(True)
        mm.sweep(S, x, w.alpha, w.q, parent=par, ancestor=anc, k=k)
        torch.cuda.synchronize()
        p = mm.profile_read()
        mm.profile_enable(False)
        ts.append({kk: v["total_ms"] / v["launches"] for kk, v in p.items()})
    ts.sort(key=lambda t: t["repulse_coarse"])
    med = ts[1]
    ms = med["repulse_coarse"]
    # kernel (a) / (d) algorithmic bytes: 4(n+1) + 12 nnz + 3 b_x n; (b_x + 4) n + b_x k
    bx = 8 if w.dim == 2 else 16
    ga = 4 * (w.n + 1) + 12 * w.S.nnz + 3 * bx * w.n
    ce = (bx + 4) * w.n + bx * k
    out = {"lib": os.path.basename(lib), "config": name, "n": w.n, "k": k, "nnz": int(w.S.nnz), "ms": ms,
           "pairs_per_s": w.n * (k - 1) / (ms / 1e3), "kernels_ms": med}
    if "gather_update" in med:
        out["gather_GBps"] = ga / (med["gather_update"] * 1e-3) / 1e9
    if "centroid" in med:
        out["centroid_GBps"] = ce / (med["centroid"] * 1e-3) / 1e9
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    cmd = sys.argv[1]
    if cmd == "build":
        from paper_1506_04383_b200 import _build

        os.makedirs(LIBS, exist_ok=True)
        _build.build(out=os.path.join(LIBS, sys.argv[2] + ".so"), extra=sys.argv[3:])
    elif cmd == "prepare":
        prepare(sys.argv[2])
    elif cmd == "time":
        for lib in sys.argv[3:]:
            subprocess.run([sys.executable, __file__, "time1", sys.argv[2], lib], check=False)
    elif cmd == "time1":
        time_one(sys.argv[2], sys.argv[3])
