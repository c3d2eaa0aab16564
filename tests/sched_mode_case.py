"""Helper for tests/test_gpu_schedule.py::test_device_loop_matches_host_loop:
run mm_layout_schedule on a few cases and save the layouts (the library reads
MM_SCHED_GRAPH once per process, so each mode runs in its own process).
Usage: MM_SCHED_GRAPH=0|1 python -m tests.sched_mode_case OUT.npz"""
import sys

import numpy as np


def main(out):
    import torch

    import paper_1506_04383_b200 as mm
    from tests.gpu_common import workload

    res = {}
    for name, h, sclap in (("cfg3_mesh64", 2, False), ("cfg2_rgg4096", 0, False), ("cfg5_grid12", 2, True)):
        w = workload(name)
        x, rep = mm.layout_schedule(mm.graph_to_device(w.graph), mm.sset_to_device(w.S), w.dim, w.q, h,
                                    mm.paper_schedule(max_final_iters=30), w.seed, n_stop=100, sclap=sclap,
                                    disc=sclap)
        torch.cuda.synchronize()
        res[f"{name}_x"] = mm.coords_from_device(x, w.dim)
        res[f"{name}_sweeps"] = np.asarray(rep["sweeps_level"])
        res[f"{name}_energy"] = np.asarray([rep["energy"]])
    np.savez(out, **res)


if __name__ == "__main__":
    main(sys.argv[1])
