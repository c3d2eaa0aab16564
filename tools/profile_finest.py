"""One finest-level Eq.(3) sweep of a multilevel config on its converged
layout, inside the NVTX range "finest", for a targeted ncu capture of kernel
(c) at the size that dominates the step:
  ncu --nvtx --nvtx-include "finest/" -k regex:k_repulse -c 1 ... python tools/profile_finest.py cfg3
The layout comes from mm_layout (h = 2), the maps from the GPU hierarchy."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1506_04383_b200 as mm  # noqa: E402
from workloads import configs  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
w = configs.make(name)
g = mm.graph_to_device(w.graph)
S = mm.sset_to_device(w.S)
x, rep = mm.layout(g, S, w.dim, w.alpha, w.q, w.h, [w.sweeps], w.seed)
H = mm.build_hierarchy(g, w.dim, w.seed)
p0 = H.level_host(0)["parent"]
p1 = H.level_host(1)["parent"]
anc = p1[p0].astype(np.int32)
k = int(H.view(2).n)
par_d = torch.from_numpy(p0.astype(np.int32)).cuda()
anc_d = torch.from_numpy(anc).cuda()
y = mm.sweep(S, x, w.alpha, w.q, parent=par_d, ancestor=anc_d, k=k)  # warm (orders, plans)
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("finest")
y = mm.sweep(S, x, w.alpha, w.q, parent=par_d, ancestor=anc_d, k=k)
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
print(name, "n", w.n, "k", k, "pairs", w.n * (k - 1))
