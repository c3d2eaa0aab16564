"""Small invocation of every entry point, for compute-sanitizer (memcheck /
racecheck / initcheck, one tool per run).  Exits non-zero on any error."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1506_04383_b200 as mm  # noqa: E402
from workloads import configs  # noqa: E402

mm.load()
w = configs.make("cfg3_mesh32")
G = mm.graph_to_device(w.graph)
S = mm.sset_to_device(w.S)
mm.validate_sset(S)
x = mm.coords_to_device(configs.random_state(w.n, 2, seed=1, scale=32.0))
y = mm.sweep(S, x, 0.01, 0.0)
H = mm.build_hierarchy(G, 2, 7, n_stop=64)
lv0, lv2 = H.level_host(0), H.level_host(2)
anc = lv0["parent"]
anc = H.level_host(1)["parent"][anc]
par = torch.from_numpy(lv0["parent"]).cuda()
y2 = mm.sweep(S, x, 0.01, 0.0, parent=par, ancestor=torch.from_numpy(anc.astype(np.int32)).cuda(), k=lv2["n"],
              stats=True)
e = mm.energy(S, y, 0.01, 0.0)
Hs = mm.build_hierarchy(G, 2, 7, n_stop=64, sclap=True)
xl, rep = mm.layout(G, S, 2, 0.01, 0.0, 2, [3], 7, n_stop=64)
xs, rep2 = mm.layout_schedule(G, S, 2, 0.0, 2, mm.paper_schedule(max_final_iters=3), 7, n_stop=64, sclap=True,
                              disc=True)
w5 = configs.make("cfg5_grid8")
G5, S5 = mm.graph_to_device(w5.graph), mm.sset_to_device(w5.S)
x5, rep5 = mm.layout(G5, S5, 3, 0.01, 0.8, 2, [2], 5, n_stop=32)
fs = mm.full_stress(G, xl)
torch.cuda.synchronize()
print("sanitize case ok", e, rep["energy"], rep2["energy"], rep5["energy"], fs[:3])
