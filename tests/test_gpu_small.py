"""-m gpu: the persistent small-level kernel (k_small.cu) that runs all the
sweeps of a level of up to 32,768 vertices (exact: 4,096) in one cooperative
launch.  mm_layout with one sweep at h = 0 goes through it for these sizes, so
its first sweep is checked against the oracle's Eq.(2) sweep; K sweeps are
checked sweep by sweep: the K-sweep launch's output against one oracle sweep
from the (K-1)-sweep launch's output (the persistent kernel is bitwise
deterministic, so that is the state its K-th sweep started from), at the
strict one-sweep bar for every K; the fused statistics against the oracle's
relative change.  The Eq.(3) path is checked the same way through
mm_sweeps with the oracle's hierarchy maps (h = 1, 2), 2-D and 3-D, q = 0 and
q = 0.8, and the launch list proves the persistent kernel ran.""" 
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
    """K = 1, 2, 3 in one launch each (ping-pong and grid barriers): the K-th
    sweep of the launch equals one oracle sweep from the (K-1)-sweep output."""
    w = workload("cfg1_grid33")
    prev = w.x0
    for K in (1, 2, 3):
        got, rep = _layout_sweeps(mm, w.S, w.x0, 2, w.alpha, w.q, K)
        assert rep["sweeps_level"] == [K]
        want = oracle.sweep_exact(w.S, prev.astype(np.float64), w.alpha, w.q)
        assert_sweep_parity(got, want, f"sweep {K} of a {K}-sweep launch")
        prev = got


def _approx_case(name, h):
    import oracle as O

    w = workload(name)
    lv = O.build_hierarchy(w.graph, seed=w.seed, n_stop=100)
    hp = min(h, len(lv) - 1)
    anc = O.ancestor(lv, 0, hp)
    # a layout-scale state: prolonged-looking clusters (parent's random spot + 1e-3 jitter)
    rng = np.random.default_rng(5)
    side = w.n ** (1.0 / w.dim)
    xc = rng.random((lv[1].n, w.dim)) * side
    x = (xc[lv[0].parent] + rng.uniform(-0.3, 0.3, (w.n, w.dim))).astype(np.float32)
    return w, lv[0].parent, anc, lv[hp].n, x


@pytest.mark.parametrize("name,h", [("cfg3_mesh64", 1), ("cfg3_mesh64", 2), ("cfg5_grid16", 1),
                                    ("cfg5_grid16", 2), ("cfg3_mesh128", 3)])
def test_small_approx_sweeps(mm, name, h):
    """Eq.(3) in the persistent kernel: sweeps 1..3 of one launch each against
    one oracle sweep_approx from the previous launch's output (1e-4 x diameter)."""
    import torch

    w, parent, anc, k, x0 = _approx_case(name, h)
    S = mm.sset_to_device(w.S)
    P = torch.from_numpy(parent.astype(np.int32)).cuda()
    A = torch.from_numpy(anc.astype(np.int32)).cuda()
    prev = x0
    for K in (1, 2, 3):
        mm.profile_reset()
        mm.profile_enable(True)
        y = mm.sweeps(S, mm.coords_to_device(x0), w.alpha, w.q, K, parent=P, ancestor=A, k=k)
        torch.cuda.synchronize()
        prof = mm.profile_read()
        mm.profile_enable(False)
        assert "small_level" in prof and "repulse_coarse" not in prof, sorted(prof)
        got = mm.coords_from_device(y, w.dim)
        want = oracle.sweep_approx(w.S, prev.astype(np.float64), w.alpha, w.q, parent, anc, k)
        assert_sweep_parity(got, want, f"{name} h={h} sweep {K}")
        prev = got


@pytest.mark.parametrize("approx", [False, True])
def test_small_coincident_points(mm, approx):
    """The persistent kernel with exactly coincident S and non-S pairs (Q6)."""
    import torch

    from tests.test_gpu_sweep import _coincident_state

    w = workload("cfg3_mesh64")
    x0 = _coincident_state(w.S, w.n, 2, seed=41)
    S = mm.sset_to_device(w.S)
    if approx:
        lv = oracle.build_hierarchy(w.graph, seed=w.seed, n_stop=100)
        anc = oracle.ancestor(lv, 0, 2)
        k = lv[2].n
        y = mm.sweeps(S, mm.coords_to_device(x0), w.alpha, w.q, 1, parent=torch.from_numpy(lv[0].parent).cuda(),
                      ancestor=torch.from_numpy(anc.astype(np.int32)).cuda(), k=k)
        want = oracle.sweep_approx(w.S, x0.astype(np.float64), w.alpha, w.q, lv[0].parent, anc, k)
    else:
        y = mm.sweeps(S, mm.coords_to_device(x0), w.alpha, w.q, 1)
        want = oracle.sweep_exact(w.S, x0.astype(np.float64), w.alpha, w.q)
    torch.cuda.synchronize()
    assert_sweep_parity(mm.coords_from_device(y, 2), want, f"small coincident approx={approx}")


def test_sweeps_tiled_path(mm):
    """mm_sweeps on a level above the small-kernel limit (the K sweeps are one
    CUDA graph of the tiled kernels, target / representative orders fixed per
    call, Q26): sweep K of a K-sweep call against one oracle sweep from the
    (K-1)-sweep call's output, at the strict bar."""
    import torch

    w, parent, anc, k, x0 = _approx_case("cfg3_mesh256", 2)
    S = mm.sset_to_device(w.S)
    P = torch.from_numpy(parent.astype(np.int32)).cuda()
    A = torch.from_numpy(anc.astype(np.int32)).cuda()
    prev = x0
    for K in (1, 2, 3):
        mm.profile_reset()
        mm.profile_enable(True)
        y = mm.sweeps(S, mm.coords_to_device(x0), w.alpha, w.q, K, parent=P, ancestor=A, k=k)
        torch.cuda.synchronize()
        prof = mm.profile_read()
        mm.profile_enable(False)
        assert "repulse_coarse" in prof and "small_level" not in prof, sorted(prof)
        got = mm.coords_from_device(y, w.dim)
        want = oracle.sweep_approx(w.S, prev.astype(np.float64), w.alpha, w.q, parent, anc, k)
        assert_sweep_parity(got, want, f"tiled sweep {K}")
        prev = got
