"""-m gpu: mm_layout_schedule (the paper's alpha schedule, and the
dynamic update mode) against the oracle's schedule driver: the
same decision trace (sweeps per level) and the final energy at alpha_min
within 1e-3 relative."""
from __future__ import annotations

import numpy as np
import pytest

import oracle
from tests.gpu_common import assert_energy, workload
from workloads import dynamic, sset

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mm():
    import torch

    import paper_1506_04383_b200 as mm

    assert torch.cuda.is_available()
    mm.load()
    return mm


def _rel(a, b):
    return abs(a - b) / max(abs(b), 1e-300)


def _sched(mm, cap):
    return mm.paper_schedule(max_final_iters=cap), oracle.paper_schedule(max_final_iters=cap)


@pytest.mark.parametrize("name,cap", [("cfg2_rgg1024", 60), ("cfg1_grid16", 30), ("cfg2_rgg4096", 40)])
def test_single_level_schedule(mm, name, cap):
    w = workload(name)
    gs, os_ = _sched(mm, cap)
    x, rep = mm.layout_schedule(None, mm.sset_to_device(w.S), 2, w.q, 0, gs, w.seed, multilevel=False,
                                x_init=mm.coords_to_device(w.x0))
    xo, eo, nl, sw = oracle.layout_schedule(w.graph, w.S, 2, w.q, 0, os_, w.seed, multilevel=False,
                                            x_init=w.x0.astype(np.float64))
    assert rep["sweeps_level"] == list(sw), (rep["sweeps_level"], list(sw))
    assert_energy(rep["energy"], eo[2], f"schedule {name} single-level")


@pytest.mark.parametrize("name,h,n_stop,cap", [("cfg3_mesh32", 0, 100, 25), ("cfg3_mesh64", 2, 200, 25),
                                               ("cfg5_grid12", 2, 100, 20), ("cfg3_mesh256", 2, 1000, 100)])
def test_multilevel_schedule(mm, name, h, n_stop, cap):
    w = workload(name)
    gs, os_ = _sched(mm, cap)
    x, rep = mm.layout_schedule(mm.graph_to_device(w.graph), mm.sset_to_device(w.S), w.dim, w.q, h, gs, w.seed,
                                n_stop=n_stop)
    xo, eo, nl, sw = oracle.layout_schedule(w.graph, w.S, w.dim, w.q, h, os_, w.seed, n_stop=n_stop)
    assert rep["levels"] == nl
    eg = oracle.energy(w.S, mm.coords_from_device(x, w.dim), 0.008, w.q)
    assert _rel(rep["energy"], eg[2]) <= 1e-4
    assert rep["sweeps_level"] == list(sw), (rep["sweeps_level"], list(sw))
    assert_energy(rep["energy"], eo[2], f"schedule {name} h={h}", levels=nl, sweeps=list(map(int, sw)),
                  rel_kernel=_rel(rep["energy"], eg[2]))


def test_dynamic_update(mm):
    """warm start of the perturbed graph Q from a layout of G, alpha_min,
    finest level only, hierarchy cut after h = 2 levels."""
    w = workload("cfg3_mesh32")
    gs, os_ = _sched(mm, 25)
    xg, _, _, _ = oracle.layout_schedule(w.graph, w.S, 2, 0.0, 2, os_, w.seed, n_stop=100)
    gq = dynamic.perturb(w.graph, 5.0, 2, seed=3)
    Sq = sset.hop2_sset(gq)
    x0 = xg.astype(np.float32)
    x, rep = mm.layout_schedule(mm.graph_to_device(gq), mm.sset_to_device(Sq), 2, 0.0, 2, gs, w.seed, dynamic=True,
                                x_init=mm.coords_to_device(x0))
    xo, eo, nl, sw = oracle.layout_schedule(gq, Sq, 2, 0.0, 2, os_, w.seed, dynamic=True,
                                            x_init=x0.astype(np.float64))
    assert rep["levels"] == nl == 3
    assert rep["sweeps_level"] == list(sw), (rep["sweeps_level"], list(sw))
    assert_energy(rep["energy"], eo[2], "schedule dynamic cfg3_mesh32")


@pytest.mark.parametrize("name,dim,n_stop,cap", [("cfg3_mesh64", 2, 100, 20), ("cfg5_grid12", 3, 100, 20),
                                                ("cfg3_mesh256", 2, 1000, 100)])
def test_schedule_sclap_disc(mm, name, dim, n_stop, cap):
    """The paper's configuration end to end: SCLaP hierarchy (R6), disc
    prolongation (R7), alpha schedule, h = 2.  mesh256's finest
    levels run on the tiled path, renumbered (Q30), with SCLaP families of
    more than two members (the gather's child-list walk)."""
    w = workload(name)
    gs, os_ = _sched(mm, cap)
    x, rep = mm.layout_schedule(mm.graph_to_device(w.graph), mm.sset_to_device(w.S), w.dim, w.q, 2, gs, w.seed,
                                n_stop=n_stop, sclap=True, disc=True)
    xo, eo, nl, sw = oracle.layout_schedule(w.graph, w.S, w.dim, w.q, 2, os_, w.seed, n_stop=n_stop, sclap=True, disc=True)
    assert rep["levels"] == nl
    eg = oracle.energy(w.S, mm.coords_from_device(x, w.dim), 0.008, w.q)
    assert _rel(rep["energy"], eg[2]) <= 1e-4
    assert rep["sweeps_level"] == list(sw), (rep["sweeps_level"], list(sw))
    assert_energy(rep["energy"], eo[2], f"schedule {name} sclap+disc", levels=nl, sweeps=list(map(int, sw)),
                  rel_kernel=_rel(rep["energy"], eg[2]))


def test_device_loop_matches_host_loop(tmp_path):
    """The device-driven schedule (one conditional-node CUDA graph per level)
    makes the host loop's decisions on the device: identical sweep counts and
    bit-identical layouts (same kernels, same order, same alpha values)."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = {}
    for mode in ("1", "0"):
        out = tmp_path / f"mode{mode}.npz"
        r = subprocess.run([sys.executable, "-m", "tests.sched_mode_case", str(out)], cwd=root,
                           env=dict(os.environ, MM_SCHED_GRAPH=mode), capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        outs[mode] = np.load(out)
    for k in outs["1"].files:
        assert np.array_equal(outs["1"][k], outs["0"][k]), k
