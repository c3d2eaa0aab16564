"""mm_energy time of a config's final layout (builder tool; MM_LIB_PATH selects the build)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1506_04383_b200 as mm  # noqa: E402
from workloads import configs  # noqa: E402

w = configs.make(sys.argv[1])
g, S = mm.graph_to_device(w.graph), mm.sset_to_device(w.S)
x, rep = mm.layout(g, S, w.dim, w.alpha, w.q, w.h, [w.sweeps], w.seed)
e = mm.energy(S, x, w.alpha, w.q)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(3):
    e = mm.energy(S, x, w.alpha, w.q)
b.record()
torch.cuda.synchronize()
print(json.dumps({"lib": os.environ.get("MM_LIB_PATH", "default"), "config": sys.argv[1], "ms": a.elapsed_time(b) / 3,
                  "energy": e[2], "layout_energy": rep["energy"]}))
