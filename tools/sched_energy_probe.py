"""Print mm_layout_schedule's energy for one multilevel schedule case (to compare
library builds via MM_LIB_PATH).  Usage: python tools/sched_energy_probe.py cfg3_mesh64 2 200 25"""
import ctypes
import os
import sys

if os.environ.get("MM_LIB_PATH"):  # older builds may lack newer symbols: stub them for this probe
    _CDLL = ctypes.CDLL

    class _Lib(_CDLL):
        def __getattr__(self, name):
            try:
                return _CDLL.__getattr__(self, name)
            except AttributeError:
                f = ctypes.CFUNCTYPE(ctypes.c_int)(lambda *a: -1)
                setattr(self, name, f)
                return f

    ctypes.CDLL = _Lib

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1506_04383_b200 as mm  # noqa: E402
from workloads import configs  # noqa: E402

name, h, n_stop, cap = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
w = configs.make(name)
gs = mm.paper_schedule(max_final_iters=cap)
for rep_i in range(2):
    x, rep = mm.layout_schedule(mm.graph_to_device(w.graph), mm.sset_to_device(w.S), w.dim, w.q, h, gs, w.seed,
                                n_stop=n_stop)
    print(os.environ.get("MM_LIB_PATH", "current"), name, h, repr(rep["energy"]), rep["sweeps_level"])
