"""-m gpu: the persistent small-level kernel (k_small.cu) that runs all the
sweeps of a level of up to 32,768 vertices (exact: 4,096) in one cooperative
launch.  mm_layout with one sweep at h = 0 goes through it for these sizes, so
its first sweep is checked against the oracle's Eq.(2) sweep; K sweeps are
checked against K oracle sweeps (Jacobi: each from the previous result); the
fused statistics against the oracle's relative change; and the Eq.(3) path
through the multilevel full runs and schedule traces of the other files."""
from __future__ import annotations

import math

import numpy as np
import pytest

import oracle
from tests import helpers as H
from tests.gpu_common import assert_sweep_parity, workload
from workloads import configs, sset

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mm():
    import torch

    import paper_1506_04383_b200 as mm

    assert torch.cuda.is_available()
    mm.load()
    return mm


def _layout_sweeps(mm, S, x, dim, alpha, q, K):
    import torch

    out, rep = mm.layout(None, mm.sset_to_device(S), dim, alpha, q, 0, [K], 1, x_init=mm.coords_to_device(x))
    torch.cuda.synchronize()
    return mm.coords_from_device(out, dim), rep


@pytest.mark.parametrize("name", ["cfg1", "cfg1_grid33"])
def test_small_exact_one_sweep(mm, name):
    w = workload(name)
    got, rep = _layout_sweeps(mm, w.S, w.x0, 2, w.alpha, w.q, 1)
    want = oracle.sweep_exact(w.S, w.x0.astype(np.float64), w.alpha, w.q)
    assert_sweep_parity(got, want, name)
    rel = oracle.relative_change(w.x0.astype(np.float64), want)
    assert abs(rep["rel_change"] - rel) <= 1e-5 * rel


@pytest.mark.parametrize("n,dim,q", [(2, 2, 0.0), (257, 3, 0.8), (1000, 2, 0.5), (4096, 2, 0.0), (3001, 3, 0.0)])
def test_small_exact_sizes(mm, n, dim, q):
    g = H.random_connected(n, n // 2 + 1, seed=n + 7)
    S = sset.hop2_sset(g) if n > 3 else H.sset_with(g, np.ones(g.nnz))
    x = configs.random_state(n, dim, seed=n, scale=math.sqrt(n))
    got, _ = _layout_sweeps(mm, S, x, dim, 0.05, q, 1)
    want = oracle.sweep_exact(S, x.astype(np.float64), 0.05, q)
    assert_sweep_parity(got, want, f"n={n} dim={dim} q={q}")


def test_small_exact_three_sweeps(mm):
    """K = 3 in one launch (ping-pong and grid barriers) vs three oracle sweeps."""
    w = workload("cfg1_grid33")
    got, rep = _layout_sweeps(mm, w.S, w.x0, 2, w.alpha, w.q, 3)
    want = w.x0.astype(np.float64)
    for _ in range(3):
        want = oracle.sweep_exact(w.S, want, w.alpha, w.q)
    assert rep["sweeps_level"] == [3]
    assert_sweep_parity(got, want, "3 sweeps", tol=3e-4)
