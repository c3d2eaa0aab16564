"""Pins for the FP64 oracle: each check is fixed by the
paper, a closed form, an invariant, a library routine or a hand derivation —
never by the oracle itself or by the CUDA path."""
from __future__ import annotations

import math

import numpy as np
import pytest
import scipy.sparse as sp
from scipy.optimize import brentq

import oracle
from tests import helpers as H
from workloads import graphs, sset


# ---------------------------------------------------------------- RNG (Q18)
def test_rng_splitmix64_reference_vector():
    """mix64 is the SplitMix64 output function: golden/splitmix64.txt."""
    g = 0x9E3779B97F4A7C15
    want = []
    with open(f"{H.GOLDEN}/splitmix64.txt") as f:
        want = [int(l, 16) for l in f if l.strip() and not l.startswith("#")]
    got = [oracle.mix64((k * g) % 2**64) for k in range(3)]
    assert got == want


def test_uniform24_range_and_exactness():
    for z in range(2000):
        k = oracle.mix64(z)
        u = oracle.uniform24(k)
        assert 0.0 <= u < 1.0
        assert u * 2**24 == float(k >> 40)  # exactly the top 24 bits


# ---------------------------------------------------------------- P1: 2-vertex path
@pytest.mark.parametrize("s0,d,w", [(1.5, 1.0, 3.0), (0.3, 2.0, 0.25), (3.1, 1.0, 1.0)])
def test_p1_two_path_period_two_orbit(s0, d, w):
    """Eq.(2) on K2 maps the separation s to (2d - |s|) s_hat, midpoint fixed
    (w cancels; no non-S pairs)."""
    g = H.path(2)
    S = H.sset_with(g, [d, d])
    S.w[:] = w
    ang = 0.7
    u = np.array([math.cos(ang), math.sin(ang)])
    mid = np.array([0.3, -1.2])
    x = np.stack([mid + 0.5 * s0 * u, mid - 0.5 * s0 * u])
    s = s0
    for k in range(6):
        x = oracle.sweep_exact(S, x, alpha=0.7, q=0.0)
        s_new = 2 * d - s
        sep = x[0] - x[1]
        np.testing.assert_allclose(sep, s_new * u, rtol=0, atol=1e-13)
        np.testing.assert_allclose(x.mean(axis=0), mid, rtol=0, atol=1e-13)
        s = abs(s_new)
        if s_new < 0:
            u = -u


def test_p1_two_path_worked_numbers():
    g = H.path(2)
    S = H.sset_with(g, [1.0, 1.0])
    x = np.array([[0.0, 0.0], [1.5, 0.0]])
    x1 = oracle.sweep_exact(S, x, 0.3, 0.0)
    np.testing.assert_allclose(x1, [[0.5, 0.0], [1.0, 0.0]], atol=1e-15)
    x2 = oracle.sweep_exact(S, x1, 0.3, 0.0)
    np.testing.assert_allclose(x2, x, atol=1e-15)


# ---------------------------------------------------------------- P2: 3-vertex path
@pytest.mark.parametrize("d,w,alpha,q", [(1, 1, 0.1, 0.0), (2, 0.25, 0.3, 0.0), (1, 1, 0.008, 0.0),
                                         (1, 1, 0.1, 0.8), (1.5, 0.5, 0.05, 0.5)])
def test_p2_three_path_fixed_point(d, w, alpha, q):
    """Collinear fixed point -L, 0, L with L = d + alpha / (w (2L)^(q+1));
    for q = 0, L = (d + sqrt(d^2 + 2 alpha / w)) / 2."""
    if q == 0.0:
        L = (d + math.sqrt(d * d + 2 * alpha / w)) / 2
    else:
        L = brentq(lambda L: L - d - alpha / (w * (2 * L) ** (q + 1)), d * 0.5, d * 10 + 10)
    g = H.path(3)
    S = H.sset_with(g, np.full(4, float(d)))
    S.w[:] = w
    x = np.array([[-L, 0.0], [0.0, 0.0], [L, 0.0]])
    # rotate and translate: the fixed point is a configuration, not coordinates
    c, s = math.cos(1.1), math.sin(1.1)
    Q = np.array([[c, -s], [s, c]])
    x = x @ Q.T + np.array([5.0, -2.0])
    y = oracle.sweep_exact(S, x, alpha, q)
    np.testing.assert_allclose(y, x, rtol=0, atol=4e-15 * (1 + abs(L)) * 10)


def test_p4_spec_worked_example_sweep():
    """golden/path3_sweep.txt (S:229 re-derived by hand)."""
    gold = H.read_golden("path3_sweep.txt")
    g = H.path(3)
    S = H.sset_with(g, np.ones(4))
    x = np.array([[0.0, 0.0], [1.0, 0.0], [2.0, 0.0]])
    y = oracle.sweep_exact(S, x, 0.008, 0.0)
    np.testing.assert_allclose(y, gold[:, 1:], rtol=0, atol=1e-15)


def test_p4_spec_worked_example_energy():
    """golden/path3_energy.txt (S:336 re-derived by hand)."""
    gold = H.read_golden("path3_energy.txt")[0]
    g = H.path(3)
    S = H.sset_with(g, np.ones(4))
    x = np.array([[0.0, 0.0], [1.0, 0.0], [2.0, 0.0]])
    e = oracle.energy(S, x, 0.008, 0.0)
    np.testing.assert_allclose(e, gold, rtol=1e-14, atol=1e-16)


# ---------------------------------------------------------------- P3: ring closed form
@pytest.mark.parametrize("n,q", [(12, 0.0), (40, 0.0), (4096, 0.0), (12, 0.8), (257, 0.8)])
def test_p3_ring_closed_form(n, q):
    """Regular n-gon of radius R, S = cycle edges, unit d, w: one sweep gives a
    regular n-gon with the same angles and radius
    R' = R cos(2pi/n) + d sin(pi/n) + (alpha/2) sum_{k=2}^{n-2} R c_k / (2 R^2 c_k)^(1+q/2),
    c_k = 1 - cos(2 pi k / n)  (= alpha (n-3) / (4R) for q = 0)."""
    R, alpha, d = 3.7, 0.05, 1.0
    th = 2 * np.pi * np.arange(n) / n + 0.3
    x = R * np.stack([np.cos(th), np.sin(th)], axis=1) + np.array([1.0, 2.0])
    g = H.cycle(n)
    S = H.sset_with(g, np.full(g.nnz, d))
    y = oracle.sweep_exact(S, x, alpha, q)
    k = np.arange(2, n - 1)
    ck = 1 - np.cos(2 * np.pi * k / n)
    if q == 0.0:
        ent = alpha * (n - 3) / (4 * R)
    else:
        ent = 0.5 * alpha * np.sum(R * ck / (2 * R * R * ck) ** (1 + q / 2))
    Rp = R * math.cos(2 * math.pi / n) + d * math.sin(math.pi / n) + ent
    want = Rp * np.stack([np.cos(th), np.sin(th)], axis=1) + np.array([1.0, 2.0])
    np.testing.assert_allclose(y, want, rtol=0, atol=1e-12 * max(1.0, Rp))


# ---------------------------------------------------------------- P5: conservation
def test_p5_weighted_sum_conserved():
    """Symmetric S: sum_i rho_i x_i is invariant under a sweep (App. B.4)."""
    g = H.random_connected(60, 80, seed=3)
    d = H.symmetric_random_d(g, 0.5, 2.0, seed=4)
    S = H.sset_with(g, d)
    rho = np.add.reduceat(S.w, S.row_ptr[:-1])
    rng = np.random.default_rng(5)
    x = rng.normal(size=(g.n, 2))
    for q in (0.0, 0.8):
        y = oracle.sweep_exact(S, x, 0.2, q)
        np.testing.assert_allclose((rho[:, None] * y).sum(0), (rho[:, None] * x).sum(0), rtol=1e-12, atol=1e-11)
    x3 = rng.normal(size=(g.n, 3))
    y3 = oracle.sweep_exact(S, x3, 0.2, 0.8)
    np.testing.assert_allclose((rho[:, None] * y3).sum(0), (rho[:, None] * x3).sum(0), rtol=1e-12, atol=1e-11)


# ---------------------------------------------------------------- P6: equivariance
def test_p6_translation_rotation_permutation():
    g = H.random_connected(50, 70, seed=7)
    S = sset.hop2_sset(g)
    rng = np.random.default_rng(8)
    x = rng.normal(size=(g.n, 2))
    y = oracle.sweep_exact(S, x, 0.1, 0.0)
    t = np.array([3.0, -7.5])
    np.testing.assert_allclose(oracle.sweep_exact(S, x + t, 0.1, 0.0), y + t, rtol=0, atol=1e-11)
    c, s = math.cos(0.9), math.sin(0.9)
    Q = np.array([[c, -s], [s, c]])
    np.testing.assert_allclose(oracle.sweep_exact(S, x @ Q.T, 0.1, 0.0), y @ Q.T, rtol=0, atol=1e-11)
    Rf = np.array([[1.0, 0.0], [0.0, -1.0]])
    np.testing.assert_allclose(oracle.sweep_exact(S, x @ Rf.T, 0.1, 0.0), y @ Rf.T, rtol=0, atol=1e-11)
    # vertex relabelling
    perm = rng.permutation(g.n)          # new id -> old id
    inv = np.argsort(perm)               # old id -> new id
    A = g.to_scipy()
    Ap = A[perm][:, perm].tocsr()
    Ap.sort_indices()
    gp = graphs.Graph(Ap.indptr.astype(np.int64), Ap.indices.astype(np.int32))
    Sp = sset.hop2_sset(gp)
    yp = oracle.sweep_exact(Sp, x[perm], 0.1, 0.0)
    np.testing.assert_allclose(yp[inv], y, rtol=0, atol=1e-12)
    # 3-D translation with q > 0
    x3 = rng.normal(size=(g.n, 3))
    y3 = oracle.sweep_exact(S, x3, 0.1, 0.8)
    t3 = np.array([1.0, 2.0, -3.0])
    np.testing.assert_allclose(oracle.sweep_exact(S, x3 + t3, 0.1, 0.8), y3 + t3, rtol=0, atol=1e-11)


# ---------------------------------------------------------------- P7: descent
def _grid4():
    return graphs.grid2d(4, 4)


@pytest.mark.parametrize("gname", ["C5", "C6", "petersen", "grid4", "path2"])
def test_p7_stress_descent_alpha0(gname):
    """alpha = 0: the stress never increases under Jacobi sweeps for symmetric S,
    w > 0 (SMACOF majorisation + signless-Laplacian PSD)."""
    g = {"C5": lambda: H.cycle(5), "C6": lambda: H.cycle(6), "petersen": H.petersen,
         "grid4": _grid4, "path2": lambda: H.path(2)}[gname]()
    for trial in range(8):
        d = H.symmetric_random_d(g, 0.5, 2.0, seed=100 + trial)
        S = H.sset_with(g, d)
        S.w[:] = H.symmetric_random_d(g, 0.5, 2.0, seed=200 + trial)
        x = np.random.default_rng(trial).normal(size=(g.n, 2)) * 2
        prev = oracle.energy(S, x, 0.0, 0.0)[0]
        for _ in range(40):
            x = oracle.sweep_exact(S, x, 0.0, 0.0)
            cur = oracle.energy(S, x, 0.0, 0.0)[0]
            assert cur <= prev * (1 + 1e-12) + 1e-14
            prev = cur


@pytest.mark.parametrize("gname", ["C5", "C6", "petersen", "grid4"])
def test_p7_energy_descent_small_alpha(gname):
    """alpha = 1e-3: M with 2 alpha (Q1) never rose on these graphs."""
    g = {"C5": lambda: H.cycle(5), "C6": lambda: H.cycle(6), "petersen": H.petersen, "grid4": _grid4}[gname]()
    alpha = 1e-3
    for trial in range(5):
        S = H.sset_with(g, np.ones(g.nnz))
        x = np.random.default_rng(50 + trial).normal(size=(g.n, 2)) * 2
        prev = oracle.energy(S, x, 2 * alpha, 0.0)[2]
        for _ in range(40):
            x = oracle.sweep_exact(S, x, alpha, 0.0)
            cur = oracle.energy(S, x, 2 * alpha, 0.0)[2]
            assert cur <= prev + 1e-12 * abs(prev) + 1e-14
            prev = cur


# ------------------------------------------- Q1: the sweep is a scaled gradient step on M_{2 alpha}
@pytest.mark.parametrize("q,dim", [(0.0, 2), (0.8, 2), (0.8, 3), (0.0, 3)])
def test_sweep_is_gradient_step_of_energy(q, dim):
    """For symmetric S:  x'_i = x_i - grad_i M_{2 alpha}(x) / (2 rho_i).
    The gradient is taken by central finite differences of oracle.energy, so a
    dropped term, sign or factor in either sweep or energy breaks this."""
    g = H.random_connected(12, 10, seed=11)
    d = H.symmetric_random_d(g, 0.7, 1.6, seed=12)
    S = H.sset_with(g, d)
    alpha = 0.3
    x = np.random.default_rng(13).normal(size=(g.n, dim)) * 1.5
    y = oracle.sweep_exact(S, x, alpha, q)
    rho = np.add.reduceat(S.w, S.row_ptr[:-1])
    grad = np.zeros_like(x)
    eps = 1e-6
    for i in range(g.n):
        for k in range(dim):
            xp = x.copy(); xp[i, k] += eps
            xm = x.copy(); xm[i, k] -= eps
            grad[i, k] = (oracle.energy(S, xp, 2 * alpha, q)[2] - oracle.energy(S, xm, 2 * alpha, q)[2]) / (2 * eps)
    np.testing.assert_allclose(y, x - grad / (2 * rho[:, None]), rtol=0, atol=2e-7)


# ---------------------------------------------------------------- P8: energy brute force
@pytest.mark.parametrize("q", [0.0, 0.8])
def test_p8_energy_bruteforce_unordered_pairs(q):
    """Eq.(1) over UNORDERED pairs with explicit set membership vs the
    oracle's per-row S_i formulation (Q4)."""
    g = H.random_connected(25, 30, seed=21)
    S = sset.hop2_sset(g)
    x = np.random.default_rng(22).normal(size=(g.n, 2))
    alpha = 0.37
    inS = {}
    for i in range(g.n):
        for e in range(S.row_ptr[i], S.row_ptr[i + 1]):
            inS[(min(i, S.col[e]), max(i, S.col[e]))] = (S.d[e], S.w[e])
    stress = ent = 0.0
    for u in range(g.n):
        for v in range(u + 1, g.n):
            r = math.dist(x[u], x[v])
            if (u, v) in inS:
                dd, ww = inS[(u, v)]
                stress += ww * (r - dd) ** 2
            else:
                ent += -math.log(r) if q == 0 else r ** (-q) / q
    got = oracle.energy(S, x, alpha, q)
    np.testing.assert_allclose(got, (stress, ent, stress + alpha * ent), rtol=1e-12)


def test_energy_closed_form_square():
    """Unit square, S = C4 edges, d = 1: stress 0, entropy = 2 * (-ln sqrt 2) = -ln 2."""
    g = H.cycle(4)
    S = H.sset_with(g, np.ones(g.nnz))
    x = np.array([[0.0, 0.0], [1.0, 0.0], [1.0, 1.0], [0.0, 1.0]])
    e = oracle.energy(S, x, 0.5, 0.0)
    np.testing.assert_allclose(e, (0.0, -math.log(2), -0.5 * math.log(2)), rtol=1e-14, atol=1e-16)


def test_energy_coincident_nonS_pair_is_error():
    g = H.path(3)
    S = H.sset_with(g, np.ones(4))
    x = np.array([[0.0, 0.0], [1.0, 0.0], [0.0, 0.0]])
    with pytest.raises(oracle.OracleError) as ei:
        oracle.energy(S, x, 0.1, 0.0)
    assert ei.value.code == oracle.OR_ECOINC


def test_sweep_rho_zero_is_error():
    g = graphs.from_edges(3, np.array([0]), np.array([1]))  # vertex 2 isolated
    S = H.sset_with(g, np.ones(g.nnz))
    with pytest.raises(oracle.OracleError) as ei:
        oracle.sweep_exact(S, np.random.default_rng(0).normal(size=(3, 2)), 0.1, 0.0)
    assert ei.value.code == oracle.OR_ERHO


def test_coincident_pairs_contribute_zero():
    """Q6: coincident S-pair gives u_ij = 0; coincident non-S pair gives r = 0."""
    g = H.path(3)
    S = H.sset_with(g, np.ones(4))
    x = np.array([[0.0, 0.0], [0.0, 0.0], [0.0, 0.0]])
    y = oracle.sweep_exact(S, x, 0.5, 0.0)
    np.testing.assert_array_equal(y, np.zeros((3, 2)))


# ---------------------------------------------------------------- P10: SMACOF / scipy
def test_p10_alpha0_is_jacobi_step_of_smacof_system():
    """alpha = 0: x' = D^-1 (W x + (diag(B 1) - B) x), B_ij = w_ij d_ij / |x_i - x_j|,
    i.e. one Jacobi step for L_w x = B(z) z (SMACOF), with scipy.sparse matvecs."""
    g = H.random_connected(200, 300, seed=31)
    d = H.symmetric_random_d(g, 0.5, 3.0, seed=32)
    S = H.sset_with(g, d)
    x = np.random.default_rng(33).normal(size=(g.n, 2)) * 3
    n = g.n
    rows = np.repeat(np.arange(n), np.diff(S.row_ptr))
    W = sp.csr_matrix((S.w, S.col, S.row_ptr), shape=(n, n))
    dist = np.linalg.norm(x[rows] - x[S.col], axis=1)
    B = sp.csr_matrix((S.w * S.d / dist, S.col, S.row_ptr), shape=(n, n))
    Dinv = 1.0 / np.asarray(W.sum(axis=1)).ravel()
    Bdiag = np.asarray(B.sum(axis=1)).ravel()
    want = Dinv[:, None] * (W @ x + Bdiag[:, None] * x - B @ x)
    np.testing.assert_allclose(oracle.sweep_exact(S, x, 0.0, 0.0), want, rtol=1e-12, atol=1e-12)


# ---------------------------------------------------------------- P9: Eq.(3)
def test_p9_identity_map_equals_eq2():
    """M = identity, nu = 1: Eq.(3) == Eq.(2)."""
    g = H.random_connected(80, 120, seed=41)
    S = sset.hop2_sset(g)
    x = np.random.default_rng(42).normal(size=(g.n, 2))
    ident = np.arange(g.n, dtype=np.int32)
    for q in (0.0, 0.8):
        a = oracle.sweep_approx(S, x, 0.2, q, ident, ident, g.n)
        b = oracle.sweep_exact(S, x, 0.2, q)
        np.testing.assert_allclose(a, b, rtol=1e-11, atol=1e-11)


def test_p9_single_cluster_equals_eq2():
    """All vertices in one cluster: the sibling sum covers every pair and the
    representative sum is empty."""
    g = H.random_connected(40, 50, seed=43)
    S = sset.hop2_sset(g)
    x = np.random.default_rng(44).normal(size=(g.n, 3))
    zero = np.zeros(g.n, dtype=np.int32)
    a = oracle.sweep_approx(S, x, 0.2, 0.8, zero, zero, 1)
    b = oracle.sweep_exact(S, x, 0.2, 0.8)
    np.testing.assert_allclose(a, b, rtol=1e-11, atol=1e-11)


def test_p9_hand_instance():
    gold = H.read_golden("eq3_hand.txt")
    g = graphs.from_edges(4, np.array([0, 1, 2]), np.array([1, 2, 3]))
    S = H.sset_with(g, np.ones(g.nnz))
    x = np.array([[0.0, 0.0], [1.0, 0.0], [0.0, 3.0], [1.0, 3.0]])
    P = np.array([0, 0, 1, 1], dtype=np.int32)
    y = oracle.sweep_approx(S, x, 0.5, 0.0, P, P, 2)
    for row in gold:
        np.testing.assert_allclose(y[int(row[0])], row[1:], rtol=0, atol=1e-14)


def test_p9_two_level_composed_map_rep_term():
    """h = 2 style maps: sibling term from P, representative term from H != P."""
    g = H.path(8)
    S = H.sset_with(g, np.ones(g.nnz))
    x = np.random.default_rng(45).normal(size=(8, 2))
    P = np.array([0, 0, 1, 1, 2, 2, 3, 3], dtype=np.int32)
    Hm = np.array([0, 0, 0, 0, 1, 1, 1, 1], dtype=np.int32)
    alpha = 0.3
    y = oracle.sweep_approx(S, x, alpha, 0.0, P, Hm, 2)
    # vertex 0: siblings {1}; rep 1 (vertices 4..7, nu = 4); minus S_0 = {1}
    xc1 = x[4:8].mean(0)
    R = (x[0] - x[1]) / np.sum((x[0] - x[1]) ** 2)
    R += 4 * (x[0] - xc1) / np.sum((x[0] - xc1) ** 2)
    R -= (x[0] - x[1]) / np.sum((x[0] - x[1]) ** 2)
    A = x[1] + (x[0] - x[1]) / np.linalg.norm(x[0] - x[1])
    np.testing.assert_allclose(y[0], A + alpha * R, rtol=1e-13)


# ---------------------------------------------------------------- P12: centroids
def test_p12_centroids_independent_recompute():
    rng = np.random.default_rng(51)
    n, k = 1000, 77
    anc = np.concatenate([np.arange(k), rng.integers(0, k, n - k)]).astype(np.int32)
    x = rng.normal(size=(n, 3))
    xc, nu = oracle.centroids(x, anc, k)
    assert nu.sum() == n
    np.testing.assert_array_equal(nu, np.bincount(anc, minlength=k))
    for c in range(3):
        np.testing.assert_allclose(xc[:, c], np.bincount(anc, weights=x[:, c], minlength=k) / nu, rtol=1e-13)


# ---------------------------------------------------------------- relative change
def test_relative_change_examples():
    assert oracle.relative_change(np.array([[1.0, 2.0]]), np.array([[1.0, 2.0]])) == 0.0
    assert oracle.relative_change(np.array([[1.0, 0.0]]), np.array([[2.0, 0.0]])) == 1.0
    np.testing.assert_allclose(oracle.relative_change(np.array([[3.0, 4.0]]), np.array([[3.0, 4.5]])), 0.1, rtol=1e-15)
