"""One mm_layout of a config (builder tool, for targeted ncu captures):
  python tools/layout_once.py cfg5 [--count]   --count prints the number of
  launches of each kernel of one layout (library profiler), so that
  `ncu -k regex:<kernel> --launch-skip <count - K>` lands on the finest level
  (the finest level runs last)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1506_04383_b200 as mm  # noqa: E402
from workloads import configs  # noqa: E402

w = configs.make(sys.argv[1])
g = mm.graph_to_device(w.graph)
S = mm.sset_to_device(w.S)
if "--count" in sys.argv:
    mm.profile_reset()
    mm.profile_enable(True)
x, rep = mm.layout(g, S, w.dim, w.alpha, w.q, w.h, [w.sweeps], w.seed)
torch.cuda.synchronize()
if "--count" in sys.argv:
    print(json.dumps({k: v["launches"] for k, v in mm.profile_read().items()}))
