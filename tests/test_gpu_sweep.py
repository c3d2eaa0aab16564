"""-m gpu: one-sweep parity of mm_sweep (Eq.(2) exact and Eq.(3) approximate)
against the FP64 oracle, through the C-ABI, plus closed forms, determinism
and edge cases."""
from __future__ import annotations

import math
import os

import numpy as np
import pytest

import oracle
from tests import helpers as H
from tests.gpu_common import assert_sweep_parity, oracle_hierarchy, sample_rows, workload
from workloads import configs, graphs, sset

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mm():
    import torch

    import paper_1506_04383_b200 as mm

    assert torch.cuda.is_available()
    mm.load()
    return mm


def _gpu_sweep(mm, S, x, alpha, q, parent=None, anc=None, k=0, stats=False):
    import torch

    Sd = mm.sset_to_device(S)
    xd = mm.coords_to_device(x)
    kw = {}
    if parent is not None:
        kw = dict(parent=torch.from_numpy(np.ascontiguousarray(parent, np.int32)).cuda(),
                  ancestor=torch.from_numpy(np.ascontiguousarray(anc, np.int32)).cuda(), k=k)
    r = mm.sweep(Sd, xd, alpha, q, stats=stats, **kw)
    torch.cuda.synchronize()
    if stats:
        y, st = r
        return mm.coords_from_device(y, x.shape[1]), st
    return mm.coords_from_device(r, x.shape[1])


# ------------------------------------------------------------------ exact, all rows
@pytest.mark.parametrize("name", ["cfg1", "cfg1_grid33", "cfg2_rgg4096", "cfg2_rgg8192"])
def test_exact_sweep_all_rows(mm, name):
    w = workload(name)
    x = w.x0.astype(np.float64)
    got = _gpu_sweep(mm, w.S, w.x0, w.alpha, w.q)
    want = oracle.sweep_exact(w.S, x, w.alpha, w.q)
    assert_sweep_parity(got, want, name)


@pytest.mark.parametrize("n,dim,q", [(1, 2, 0.0), (2, 2, 0.0), (3, 3, 0.8), (255, 2, 0.0), (257, 2, 0.8),
                                     (1023, 3, 0.0), (1025, 3, 0.8), (4097, 2, 0.5)])
def test_exact_sweep_ragged_sizes(mm, n, dim, q):
    """Sizes around the 256-target tile and 1024-target CTA boundaries."""
    if n == 1:
        g = graphs.Graph(np.zeros(2, np.int64), np.zeros(0, np.int32))
        pytest.skip("n = 1 has an empty S row: rho = 0 is invalid input (Q22)")
    g = H.random_connected(n, n // 2 + 1, seed=n)
    S = sset.hop2_sset(g) if n > 3 else H.sset_with(g, np.ones(g.nnz))
    x = configs.random_state(n, dim, seed=n + 1, scale=math.sqrt(n))
    got = _gpu_sweep(mm, S, x, 0.05, q)
    want = oracle.sweep_exact(S, x.astype(np.float64), 0.05, q)
    assert_sweep_parity(got, want, f"n={n} dim={dim} q={q}")


def test_exact_sweep_cfg2_full_sampled_rows(mm):
    """configs[1] at full size (n = 65,428 LCC), launch configuration of bench.py,
    oracle evaluated on 2,048 sampled rows (plus the max-|S_i| rows)."""
    w = workload("cfg2")
    got = _gpu_sweep(mm, w.S, w.x0, w.alpha, w.q)
    rl = w.S.row_lengths()
    rows = sample_rows(w.n, 2048, seed=5, extra=np.argsort(rl)[-8:])
    want = oracle.sweep_exact(w.S, w.x0.astype(np.float64), w.alpha, w.q, rows=rows)
    assert_sweep_parity(got[rows], want, "cfg2 sampled")


def test_exact_sweep_3d_q08(mm):
    w = workload("cfg5_grid12")
    x = configs.random_state(w.n, 3, seed=3, scale=12.0)
    got = _gpu_sweep(mm, w.S, x, w.alpha, w.q)
    want = oracle.sweep_exact(w.S, x.astype(np.float64), w.alpha, w.q)
    assert_sweep_parity(got, want, "grid12^3 q=0.8")


# ------------------------------------------------------------------ closed form at scale
@pytest.mark.parametrize("n,q", [(65536, 0.0), (4099, 0.8)])
def test_ring_closed_form(mm, n, q):
    """one sweep of a regular n-gon (S = ring edges) gives the n-gon of
    radius R' = R cos(2pi/n) + d sin(pi/n) + (alpha/2) sum_k R c_k/(2R^2 c_k)^(1+q/2);
    exercises the full O(n^2) kernel against an FP64 formula (no oracle)."""
    R, alpha, d = 0.5 * n / math.pi, 0.05, 1.0
    th = 2 * np.pi * np.arange(n) / n
    x = (R * np.stack([np.cos(th), np.sin(th)], axis=1)).astype(np.float32)
    g = H.cycle(n)
    S = H.sset_with(g, np.full(g.nnz, d))
    got = _gpu_sweep(mm, S, x, alpha, q)
    k = np.arange(2, n - 1)
    ck = 1 - np.cos(2 * np.pi * k / n)
    ent = alpha * (n - 3) / (4 * R) if q == 0 else 0.5 * alpha * np.sum(R * ck / (2 * R * R * ck) ** (1 + q / 2))
    xr = x.astype(np.float64)
    Rin = np.linalg.norm(xr, axis=1)  # exact radius of the FP32 input points
    Rp = Rin * math.cos(2 * math.pi / n) + d * math.sin(math.pi / n) + ent
    want = (Rp / Rin)[:, None] * xr
    assert_sweep_parity(got, want, f"ring n={n}")


# ------------------------------------------------------------------ Eq.(3)
@pytest.mark.parametrize("name,h", [("cfg3_mesh64", 2), ("cfg3_mesh64", 1), ("cfg5_grid16", 2),
                                    ("cfg4_cl20000", 2), ("cfg3_mesh128", 3)])
def test_approx_sweep_all_rows(mm, name, h):
    w = workload(name)
    lv = oracle_hierarchy(name)
    L = len(lv) - 1
    hp = min(h, L)
    anc = oracle.ancestor(lv, 0, hp)
    k = lv[hp].n
    x = configs.random_state(w.n, w.dim, seed=11, scale=math.sqrt(w.n))
    got = _gpu_sweep(mm, w.S, x, w.alpha, w.q, lv[0].parent, anc, k)
    want = oracle.sweep_approx(w.S, x.astype(np.float64), w.alpha, w.q, lv[0].parent, anc, k)
    assert_sweep_parity(got, want, f"{name} h={h}")


@pytest.mark.parametrize("name,rows", [("cfg3", 4096), ("cfg4", 2048), ("cfg5", 1024)])
def test_approx_sweep_full_size_sampled(mm, name, rows):
    """Full-size configs[2..4]: the GPU sweeps every vertex; the oracle
    evaluates sampled rows with its own hierarchy (maps are bit-identical,
    test_gpu_hierarchy)."""
    w = workload(name)
    lv = oracle_hierarchy(name)
    anc = oracle.ancestor(lv, 0, 2)
    k = lv[2].n
    x = configs.random_state(w.n, w.dim, seed=12, scale=w.n ** (1.0 / w.dim))
    got = _gpu_sweep(mm, w.S, x, w.alpha, w.q, lv[0].parent, anc, k)
    rl = w.S.row_lengths()
    r = sample_rows(w.n, rows, seed=13, extra=np.argsort(rl)[-4:])
    want = oracle.sweep_approx(w.S, x.astype(np.float64), w.alpha, w.q, lv[0].parent, anc, k, rows=r)
    assert_sweep_parity(got[r], want, f"{name} sampled")


def _structured_state(name, lv, dim, disc: bool, offset: float):
    """A clustered layout built only from the oracle's own steps: the level-2
    clusters at a seeded box position (Q14's scale), prolonged to level 1 and
    level 0 (Q15 jitter, or the paper's disc P:240-242), then shifted by
    `offset` in every coordinate (cfg4's converged layouts sit at 885-1140,
    where FP32 differences to a centroid cancel: Q24, Q28)."""
    n2 = lv[2].n
    x = oracle.init_box(n2, dim, float(lv[0].n) ** (1.0 / dim), seed=21, level=2)
    for l in (1, 0):
        if disc:
            x = oracle.prolong_disc(lv[l].parent, x, lv[l + 1].c, seed=21, level=l)
        else:
            x = oracle.prolong(lv[l].parent, x, seed=21, level=l)
    return (x + offset).astype(np.float32)


@pytest.mark.parametrize("name,disc,rows", [("cfg4", True, 2048), ("cfg4", False, 1024), ("cfg5", True, 512)])
def test_approx_sweep_full_size_structured(mm, name, disc, rows):
    """Full-size Eq.(3) sweep from a clustered, offset state (not a random one):
    representatives sit among their members, most tiles are near a warp's
    targets, and the centroid differences need the hi/lo split (Q24-Q28)."""
    w = workload(name)
    lv = oracle_hierarchy(name)
    anc = oracle.ancestor(lv, 0, 2)
    k = lv[2].n
    x = _structured_state(name, lv, w.dim, disc, 1000.0)
    got = _gpu_sweep(mm, w.S, x, w.alpha, w.q, lv[0].parent, anc, k)
    rl = w.S.row_lengths()
    r = sample_rows(w.n, rows, seed=14, extra=np.argsort(rl)[-4:])
    want = oracle.sweep_approx(w.S, x.astype(np.float64), w.alpha, w.q, lv[0].parent, anc, k, rows=r)
    assert_sweep_parity(got[r], want, f"{name} structured disc={disc} sampled")


def _coincident_state(S, n, dim, seed, count=25):
    """A random state where `count` S pairs and `count` non-S pairs coincide
    exactly (x_j := x_i bit for bit): Q6, both sides take such a pair's unit
    vector and r-value as 0."""
    rng = np.random.default_rng(seed)
    x = configs.random_state(n, dim, seed=seed, scale=math.sqrt(n))
    rp, col = S.row_ptr, S.col
    used = set()
    for i in rng.choice(n, count, replace=False):
        j = int(col[rp[i] + rng.integers(0, rp[i + 1] - rp[i])])
        if i in used or j in used:
            continue
        x[j] = x[i]
        used.update((int(i), j))
    placed = 0
    while placed < count:
        a, b = (int(v) for v in rng.choice(n, 2, replace=False))
        if a in used or b in used or b in set(col[rp[a]:rp[a + 1]].tolist()):
            continue
        x[b] = x[a]
        used.update((a, b))
        placed += 1
    return x


@pytest.mark.parametrize("dim,q", [(2, 0.0), (3, 0.8), (2, 0.5), (3, 0.0)])
def test_exact_sweep_coincident_points(mm, dim, q):
    """Exactly coincident S pairs and non-S pairs (Q6): finite output equal to
    the oracle's.  Run by every kernel (b) variant (test_gpu_sym.py forces
    each)."""
    n = 3001
    g = H.random_connected(n, n // 2 + 1, seed=31)
    S = sset.hop2_sset(g)
    x = _coincident_state(S, n, dim, seed=32)
    got = _gpu_sweep(mm, S, x, 0.05, q)
    want = oracle.sweep_exact(S, x.astype(np.float64), 0.05, q)
    assert_sweep_parity(got, want, f"coincident dim={dim} q={q}")


@pytest.mark.parametrize("name,q", [("cfg3_mesh64", 0.0), ("cfg5_grid16", 0.8), ("cfg3_mesh128", 0.5)])
def test_approx_sweep_coincident_points(mm, name, q):
    """Kernel (c) + (a) with exactly coincident S pairs and non-S pairs (Q6)."""
    w = workload(name)
    lv = oracle_hierarchy(name)
    anc = oracle.ancestor(lv, 0, 2)
    k = lv[2].n
    x = _coincident_state(w.S, w.n, w.dim, seed=33)
    got = _gpu_sweep(mm, w.S, x, w.alpha, q, lv[0].parent, anc, k)
    want = oracle.sweep_approx(w.S, x.astype(np.float64), w.alpha, q, lv[0].parent, anc, k)
    assert_sweep_parity(got, want, f"{name} coincident q={q}")


def test_approx_identity_map_equals_exact(mm):
    """P:281 on the GPU: M = identity makes Eq.(3) equal Eq.(2)."""
    w = workload("cfg2_rgg4096")
    ident = np.arange(w.n, dtype=np.int32)
    a = _gpu_sweep(mm, w.S, w.x0, w.alpha, w.q, ident, ident, w.n)
    b = _gpu_sweep(mm, w.S, w.x0, w.alpha, w.q)
    assert_sweep_parity(a, b.astype(np.float64), "identity vs exact")


def test_approx_single_cluster_equals_exact(mm):
    w = workload("cfg1")
    zero = np.zeros(w.n, dtype=np.int32)
    a = _gpu_sweep(mm, w.S, w.x0, w.alpha, w.q, zero, zero, 1)
    want = oracle.sweep_exact(w.S, w.x0.astype(np.float64), w.alpha, w.q)
    assert_sweep_parity(a, want, "single cluster")


# ------------------------------------------------------------------ properties
def test_determinism_bitwise(mm):
    w = workload("cfg2_rgg8192")
    a = _gpu_sweep(mm, w.S, w.x0, w.alpha, w.q)
    b = _gpu_sweep(mm, w.S, w.x0, w.alpha, w.q)
    assert np.array_equal(a, b)
    w3 = workload("cfg3_mesh64")
    lv = oracle_hierarchy("cfg3_mesh64")
    anc = oracle.ancestor(lv, 0, 2)
    x = configs.random_state(w3.n, 2, seed=1, scale=64.0)
    c = _gpu_sweep(mm, w3.S, x, w3.alpha, w3.q, lv[0].parent, anc, lv[2].n)
    d = _gpu_sweep(mm, w3.S, x, w3.alpha, w3.q, lv[0].parent, anc, lv[2].n)
    assert np.array_equal(c, d)


def test_translation_invariance_gpu(mm):
    w = workload("cfg1")
    a = _gpu_sweep(mm, w.S, w.x0, w.alpha, w.q)
    t = np.array([3.0, -2.0], dtype=np.float32)
    b = _gpu_sweep(mm, w.S, w.x0 + t, w.alpha, w.q)
    assert_sweep_parity(b - t, a.astype(np.float64), "translation")


def test_sweep_stats(mm):
    """Relative change and stress from the fused reduction (e)."""
    w = workload("cfg2_rgg4096")
    got, st = _gpu_sweep(mm, w.S, w.x0, w.alpha, w.q, stats=True)
    x = w.x0.astype(np.float64)
    want = oracle.sweep_exact(w.S, x, w.alpha, w.q)
    rc = oracle.relative_change(x, want)
    assert st["flags"] == 0
    assert abs(math.sqrt(st["dx2"] / st["x2"]) - rc) <= 1e-4 * rc
    stress = oracle.energy(w.S, x, 0.0, 0.0)[0]
    assert abs(st["stress"] - stress) <= 1e-4 * stress


def test_nonfinite_flag(mm):
    w = workload("cfg1")
    x = w.x0.copy()
    x[5, 0] = np.nan
    _, st = _gpu_sweep(mm, w.S, x, w.alpha, w.q, stats=True)
    assert st["flags"] & 1


def test_validate_sset(mm):
    """mm_validate_sset flags each documented input error (MM_ERR_INVALID_INPUT)."""
    import torch

    w = workload("cfg1")
    mm.validate_sset(mm.sset_to_device(w.S))  # valid
    cases = []
    S = mm.sset_to_device(w.S)
    S.d[3] = 0.0
    cases.append((S, "d <= 0"))
    S = mm.sset_to_device(w.S)
    S.w[5] = float("nan")
    cases.append((S, "w < 0"))
    S = mm.sset_to_device(w.S)
    S.col[7] = w.n + 3
    cases.append((S, "out of range"))
    S = mm.sset_to_device(w.S)
    S.col[int(w.S.row_ptr[2])] = 2
    cases.append((S, "self entry"))
    S = mm.sset_to_device(w.S)
    S.w[int(w.S.row_ptr[9]):int(w.S.row_ptr[10])] = 0.0
    cases.append((S, "rho_i <= 0"))
    for S, what in cases:
        with pytest.raises(mm.MMError) as ei:
            mm.validate_sset(S)
        assert ei.value.status == -2 and what in str(ei.value), (what, str(ei.value))
    torch.cuda.synchronize()


def test_two_path_orbit_gpu(mm):
    """P1 on the GPU: K2 maps the separation s to (2d - |s|) s_hat, midpoint fixed."""
    g = H.path(2)
    S = H.sset_with(g, [1.0, 1.0])
    x = np.array([[0.0, 0.0], [1.5, 0.0]], dtype=np.float32)
    y = _gpu_sweep(mm, S, x, 0.3, 0.0)
    np.testing.assert_allclose(y, [[0.5, 0.0], [1.0, 0.0]], atol=1e-6)
    z = _gpu_sweep(mm, S, y.astype(np.float32), 0.3, 0.0)
    np.testing.assert_allclose(z, x, atol=1e-6)


def test_exact_sweep_3d_q0(mm):
    w = workload("cfg5_grid12")
    x = configs.random_state(w.n, 3, seed=8, scale=12.0)
    got = _gpu_sweep(mm, w.S, x, w.alpha, 0.0)
    want = oracle.sweep_exact(w.S, x.astype(np.float64), w.alpha, 0.0)
    assert_sweep_parity(got, want, "grid12^3 q=0")


def test_empty_and_degenerate_inputs_rejected(mm):
    import ctypes

    from paper_1506_04383_b200 import mulment

    L = mm.load()
    s = mulment.mm_sset(0, 0, 0x1000, None, None, None)
    rc = L.mm_sweep(ctypes.byref(s), 2, 0.1, 0.0, None, 0x5000, 0x6000, None, None, 0, None)
    assert rc == mulment.MM_ERR_INVALID_ARGUMENT
    out = (ctypes.c_double * 4)()
    g = mulment.mm_graph(0, 0, 0x1000, None, None)
    assert L.mm_full_stress(ctypes.byref(g), 2, 0x5000, out, None) == mulment.MM_ERR_INVALID_ARGUMENT
    # approximate sweep with k out of range
    w = workload("cfg1")
    import torch
    Sd = mm.sset_to_device(w.S)
    xd = mm.coords_to_device(w.x0)
    par = torch.zeros(w.n, dtype=torch.int32, device="cuda")
    with pytest.raises(mm.MMError):
        mm.sweep(Sd, xd, 0.1, 0.0, parent=par, ancestor=par, k=w.n + 1)


@pytest.mark.parametrize("name,approx", [("cfg2", False), ("cfg3_mesh64", True)])
def test_caller_workspace_bitwise(mm, name, approx):
    """mm_sweep with caller-provided scratch (mm_sweep_workspace bytes) equals the
    library-allocated path bit for bit (exact: the symmetric kernel at cfg2)."""
    import torch

    w = workload(name)
    x = w.x0 if w.x0 is not None else configs.random_state(w.n, w.dim, seed=2, scale=64.0)
    S = mm.sset_to_device(w.S)
    xd = mm.coords_to_device(x)
    kw, k = {}, 0
    if approx:
        lv = oracle_hierarchy(name)
        anc = oracle.ancestor(lv, 0, 2)
        k = lv[2].n
        kw = dict(parent=torch.from_numpy(lv[0].parent.astype(np.int32)).cuda(),
                  ancestor=torch.from_numpy(anc.astype(np.int32)).cuda(), k=k)
    a = mm.sweep(S, xd, w.alpha, w.q, **kw)
    ws = torch.empty(mm.sweep_workspace(w.n, w.dim, k), dtype=torch.uint8, device="cuda")
    b = mm.sweep(S, xd, w.alpha, w.q, workspace=ws, **kw)
    torch.cuda.synchronize()
    assert torch.equal(a, b)
    with pytest.raises(mm.MMError):
        mm.sweep(S, xd, w.alpha, w.q, workspace=ws[:64], **kw)


@pytest.mark.parametrize("n,q", [(30001, 0.8), (25000, 0.0)])
def test_exact_sweep_3d_symmetric_sampled(mm, n, q):
    """3-D exact sweeps above the symmetric kernel's threshold (n >~ 21K), so
    the default path takes it; 1,024 sampled rows against the oracle.  Under a
    forced kernel (MM_SYM, test_gpu_sym.py) the same rows check that kernel."""
    if "MM_SYM" not in os.environ:
        assert mm.exact_kernel_variant(n, 3) == 1
    g = H.random_connected(n, n // 2 + 1, seed=n)
    S = sset.hop2_sset(g)
    x = configs.random_state(n, 3, seed=n + 3, scale=n ** (1 / 3))
    got = _gpu_sweep(mm, S, x, 0.05, q)
    rows = sample_rows(n, 1024, seed=11)
    want = oracle.sweep_exact(S, x.astype(np.float64), 0.05, q, rows=rows)
    assert_sweep_parity(got[rows], want, f"3-D n={n} q={q}")


@pytest.mark.parametrize("offset", [0.0, 2.0e4])
def test_approx_far_tiles_structured_layout(mm, offset):
    """Eq.(3) on a layout with spatially compact clusters (the mesh drawn on its
    grid, jittered), so that with the far-tile path on (MM_FAR_PAIRS=1 in
    test_gpu_coarse_modes.py; off at this size by default) most (warp, tile)
    pairs take kernel (c)'s lo-free far path (Q27); translated by
    `offset` the frame origin (Q28) moves to the layout.  All rows against the
    oracle."""
    w = workload("cfg3_mesh128")
    lv = oracle_hierarchy("cfg3_mesh128")
    anc = oracle.ancestor(lv, 0, 2)
    k = lv[2].n
    side = int(round(math.sqrt(w.n)))
    ids = np.arange(w.n)
    rng = np.random.default_rng(5)
    x = np.stack([ids % side, ids // side], axis=1).astype(np.float64)
    x += rng.uniform(-0.2, 0.2, size=x.shape) + offset
    x = x.astype(np.float32)
    got = _gpu_sweep(mm, w.S, x, w.alpha, w.q, lv[0].parent, anc, k)
    want = oracle.sweep_approx(w.S, x.astype(np.float64), w.alpha, w.q, lv[0].parent, anc, k)
    assert_sweep_parity(got, want, f"structured offset={offset}")
