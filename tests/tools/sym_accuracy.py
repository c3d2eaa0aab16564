"""One exact sweep, GPU vs FP64 oracle, for the kernel selected by MM_SYM
(run once per mode): max |x_gpu - x_oracle| / bbox diameter and the RMS error.
Usage: MM_SYM=2|0 python tests/tools/sym_accuracy.py cfg2_rgg8192 cfg2_rgg16384"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import oracle  # noqa: E402  (tool: compares against the test oracle)
import paper_1506_04383_b200 as mm  # noqa: E402
from workloads import configs  # noqa: E402

for name in sys.argv[1:]:
    w = configs.make(name)
    S = mm.sset_to_device(w.S)
    y = mm.sweep(S, mm.coords_to_device(w.x0), w.alpha, w.q)
    torch.cuda.synchronize()
    got = mm.coords_from_device(y, w.dim).astype(np.float64)
    want = oracle.sweep_exact(w.S, w.x0.astype(np.float64), w.alpha, w.q)
    diam = float(np.linalg.norm(want.max(0) - want.min(0)))
    e = np.abs(got - want)
    print(name, "MM_SYM", os.environ.get("MM_SYM", "1"), "variant", mm.exact_kernel_variant(w.n, w.dim),
          "max/diam %.3e rms/diam %.3e" % (e.max() / diam, np.sqrt((e ** 2).mean()) / diam), flush=True)
