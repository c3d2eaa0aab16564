"""Diagnose Eq.(3) parity: worst rows of GPU vs oracle with an FP64 numpy
decomposition of the entropy term (debug tool, not part of the product)."""
import math
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import oracle  # noqa: E402
import paper_1506_04383_b200 as mm  # noqa: E402
from workloads import configs  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg3_mesh128"
h = int(sys.argv[2]) if len(sys.argv) > 2 else 3
w = configs.make(name)
lv = oracle.build_hierarchy(w.graph, seed=w.seed, n_stop=1000)
hp = min(h, len(lv) - 1)
anc = oracle.ancestor(lv, 0, hp)
k = lv[hp].n
P = lv[0].parent
x = configs.random_state(w.n, w.dim, seed=11, scale=math.sqrt(w.n)).astype(np.float32)
S = mm.sset_to_device(w.S)
y = mm.sweep(S, mm.coords_to_device(x), w.alpha, w.q, parent=torch.from_numpy(P).cuda(),
             ancestor=torch.from_numpy(anc).cuda(), k=k)
got = mm.coords_from_device(y, w.dim)
xd = x.astype(np.float64)
want = oracle.sweep_approx(w.S, xd, w.alpha, w.q, P, anc, k)
err = np.abs(got - want).max(axis=1)
diam = np.linalg.norm(want.max(0) - want.min(0))
print("levels", [l.n for l in lv], "k", k, "max err", err.max(), "diam", diam)
xc, nu = oracle.centroids(xd, anc, k)
for i in np.argsort(err)[-5:][::-1]:
    rho = w.S.w[w.S.row_ptr[i]:w.S.row_ptr[i + 1]].sum()
    sib = [j for j in np.nonzero(P == P[i])[0] if j != i]
    dv = xd[i] - xc
    r2 = (dv ** 2).sum(1)
    mask = np.arange(k) != anc[i]
    rep = (nu[mask, None] * dv[mask] / r2[mask, None]).sum(0)
    print(f"row {i}: err {err[i]:.3e} gpu {got[i]} oracle {want[i]} rho {rho:.3f} sib {sib} H {anc[i]} nu {nu[anc[i]]}")
    print(f"   min rep dist {np.sqrt(r2[mask].min()):.3e} rep-sum {rep} |x_i - x'_H| {np.sqrt(r2[anc[i]]):.3e}")
    for j in sib:
        print(f"   sibling {j} dist {np.linalg.norm(xd[i] - xd[j]):.3e} in S: {j in set(w.S.col[w.S.row_ptr[i]:w.S.row_ptr[i+1]])}")
    nb = w.S.col[w.S.row_ptr[i]:w.S.row_ptr[i + 1]]
    print(f"   min S dist {np.linalg.norm(xd[i] - xd[nb], axis=1).min():.3e}")
