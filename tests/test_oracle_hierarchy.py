"""Pins for the oracle hierarchy, prolongation and driver."""
from __future__ import annotations

import numpy as np
import pytest
import scipy.sparse as sp

import oracle
from tests import helpers as H
from workloads import configs, graphs


def _check_level_pair(fine: oracle.Level, coarse: oracle.Level):
    P = fine.parent
    n, k = fine.n, coarse.n
    # parent surjective, clusters of size 1 or 2 (a matching)
    sizes = np.bincount(P, minlength=k)
    assert sizes.min() >= 1 and sizes.max() <= 2 and sizes.shape[0] == k
    # node weights conserved per cluster
    np.testing.assert_array_equal(np.bincount(P, weights=fine.c, minlength=k).astype(np.int64), coarse.c)
    # coarse omega = brute-force crossing sums  Pm^T A Pm  off the diagonal
    A = sp.csr_matrix((fine.omega.astype(np.float64), fine.col, fine.row_ptr), shape=(n, n))
    Pm = sp.csr_matrix((np.ones(n), (np.arange(n), P)), shape=(n, k))
    C = (Pm.T @ A @ Pm).tocsr()
    C.setdiag(0)
    C.eliminate_zeros()
    C.sort_indices()
    np.testing.assert_array_equal(C.indptr, coarse.row_ptr)
    np.testing.assert_array_equal(C.indices, coarse.col)
    np.testing.assert_array_equal(C.data.astype(np.int64), coarse.omega)
    # every matched pair is an edge of the fine graph
    rows = np.repeat(np.arange(n), np.diff(fine.row_ptr))
    edges = set(zip(rows.tolist(), fine.col.tolist()))
    for cl in np.nonzero(sizes == 2)[0][:2000]:
        a, b = np.nonzero(P == cl)[0]
        assert (a, b) in edges
    # coarse ids are ranks of leaders min(u, mate(u)) in ascending order
    leaders = np.array([np.nonzero(P == c)[0].min() for c in range(min(k, 500))])
    assert np.all(np.diff(leaders) > 0)


def _maximal(fine: oracle.Level) -> bool:
    P = fine.parent
    sizes = np.bincount(P)
    single = sizes[P] == 1
    rows = np.repeat(np.arange(fine.n), np.diff(fine.row_ptr))
    return not np.any(single[rows] & single[fine.col])


@pytest.mark.parametrize("name", ["cfg3_mesh64", "cfg5_grid16", "cfg1"])
def test_p11_hierarchy_invariants(name):
    w = configs.make(name)
    lv = oracle.build_hierarchy(w.graph, seed=w.seed, n_stop=100)
    assert len(lv) >= 2
    for l in range(len(lv) - 1):
        _check_level_pair(lv[l], lv[l + 1])
        assert lv[l + 1].n <= 0.9 * lv[l].n
        if lv[l].rounds < 64:
            assert _maximal(lv[l])
    assert lv[-1].n <= 100 or lv[-1].parent is None
    assert lv[0].c.sum() == lv[-1].c.sum() == w.n


def test_p11_hierarchy_chung_lu_small():
    w = configs.make("cfg4_cl20000")
    lv = oracle.build_hierarchy(w.graph, seed=w.seed, n_stop=1000)
    for l in range(len(lv) - 1):
        _check_level_pair(lv[l], lv[l + 1])
    assert lv[-1].n <= 1000


def test_p11_triangle_hand_instance():
    """Triangle a,b,c with omega(a,b)=1, (a,c)=2, (b,c)=3, unit c: every vertex's
    best is its heaviest edge; b and c pick each other, a stays single.
    Coarse: {a} (id 0, c=1), {b,c} (id 1, c=2), one edge with omega 1+2 = 3
    (the crossing edges)."""
    g = graphs.from_edges(3, np.array([0, 0, 1]), np.array([1, 2, 2]))
    # CSR rows: 0:[1,2] 1:[0,2] 2:[0,1]
    om = np.array([1, 2, 1, 3, 2, 3], dtype=np.int64)
    lv = oracle.build_hierarchy(g, seed=1, n_stop=1, omega=om)
    assert lv[0].parent.tolist() == [0, 1, 1]
    assert lv[1].c.tolist() == [1, 2]
    assert lv[1].col.tolist() == [1, 0] and lv[1].omega.tolist() == [3, 3]


def test_p11_rating_normalised_by_weights():
    """Rating omega / (c_u c_v): with omega equal, the lighter neighbour wins."""
    # star: centre 0, leaves 1 (c=5), 2 (c=1), 3 (c=3); unit omega
    g = graphs.from_edges(4, np.array([0, 0, 0]), np.array([1, 2, 3]))
    c = np.array([1, 5, 1, 3], dtype=np.int64)
    lv = oracle.build_hierarchy(g, seed=9, n_stop=1, c=c)
    P = lv[0].parent
    assert P[0] == P[2] and P[1] != P[0] and P[3] != P[0]


def test_hierarchy_deterministic_and_seed_dependent():
    w = configs.make("cfg3_mesh64")
    a = oracle.build_hierarchy(w.graph, seed=5)
    b = oracle.build_hierarchy(w.graph, seed=5)
    c = oracle.build_hierarchy(w.graph, seed=6)
    assert all(np.array_equal(x.parent, y.parent) for x, y in zip(a[:-1], b[:-1]))
    assert not np.array_equal(a[0].parent, c[0].parent)


def test_p13_prolongation_bounds_and_rng():
    rng = np.random.default_rng(3)
    parent = rng.integers(0, 50, 400).astype(np.int32)
    xc = rng.normal(size=(50, 3))
    x = oracle.prolong(parent, xc, seed=77, level=2)
    dev = x - xc[parent]
    assert np.all(np.abs(dev) <= 1e-3)
    # the jitter is 1e-3 (2U - 1) with U the counter RNG of (seed, JITTER, level, u*dim + k)
    u, k = 123, 2
    U = oracle.uniform24(oracle.key_vertex(77, oracle.TAG_JITTER, 2, u, 3, k))
    assert dev[u, k] == pytest.approx(1e-3 * (2 * U - 1), abs=1e-15)
    # different levels -> different draws
    x2 = oracle.prolong(parent, xc, seed=77, level=3)
    assert not np.array_equal(x, x2)


TAG_DISC = 0x44495343  # oracle/mm_oracle.h OR_TAG_DISC


@pytest.mark.parametrize("dim", [2, 3])
def test_prolong_disc_laws(dim):
    """The paper's disc prolongation: "a random position in a circle
    around P with radius r := sqrt(c(v'))", "an angle uniformly at random in
    [0, 2 pi] and a distance to P uniformly at random in [0, r]" (dim 3, R7:
    radius c^(1/3), direction uniform on the sphere).  Pinned by the laws the
    sentence states, not by the oracle's formula: every point within r of its
    parent; distance / r uniform on [0, 1] (mean 1/2, not the 2/3 of an
    area-uniform disc); direction uniform (mean 0, second moment 1/dim per
    axis, equal quadrant counts)."""
    rng = np.random.default_rng(11)
    nc, n = 64, 40000
    parent = rng.integers(0, nc, n).astype(np.int32)
    xc = rng.normal(size=(nc, dim)) * 50.0
    c = rng.integers(1, 40, nc).astype(np.int64)
    x = oracle.prolong_disc(parent, xc, c, seed=5, level=1)
    dev = x - xc[parent]
    r = c[parent].astype(np.float64) ** (1.0 / dim)
    dist = np.linalg.norm(dev, axis=1)
    assert np.all(dist <= r * (1 + 1e-12))
    t = dist / r
    assert abs(t.mean() - 0.5) < 0.01
    assert abs((t ** 2).mean() - 1.0 / 3.0) < 0.01
    for q in (0.25, 0.5, 0.75):  # CDF of U[0, 1]
        assert abs((t <= q).mean() - q) < 0.01
    u = dev / np.maximum(dist, 1e-300)[:, None]
    assert np.all(np.abs(u.mean(axis=0)) < 0.02)
    assert np.all(np.abs((u ** 2).mean(axis=0) - 1.0 / dim) < 0.01)
    quad = (u[:, 0] > 0).astype(int) * 2 + (u[:, 1] > 0)
    assert np.all(np.abs(np.bincount(quad, minlength=4) / n - 0.25) < 0.01)


def test_prolong_disc_hand_point_and_keys():
    """Polar geometry by hand: with the draws U0, U1 of the pinned RNG, the
    vertex lies at distance r U1 from its parent at angle 2 pi U0 (P:242:
    "used as a polar coordinate for v with respect to the origin P"); the
    draws are keyed by (seed, DISC tag, fine level, vertex)."""
    parent = np.zeros(300, dtype=np.int32)
    xc = np.array([[10.0, -4.0]])
    c = np.array([9], dtype=np.int64)  # r = 3
    x = oracle.prolong_disc(parent, xc, c, seed=9, level=4)
    for u in (0, 17, 299):
        U0 = oracle.uniform24(oracle.key_vertex(9, TAG_DISC, 4, u, 3, 0))
        U1 = oracle.uniform24(oracle.key_vertex(9, TAG_DISC, 4, u, 3, 1))
        d = x[u] - xc[0]
        assert np.hypot(*d) == pytest.approx(3.0 * U1, rel=1e-12)
        if U1 > 1e-6:
            ang = np.arctan2(d[1], d[0]) % (2 * np.pi)
            assert ang == pytest.approx(2 * np.pi * U0, abs=1e-9)
    x2 = oracle.prolong_disc(parent, xc, c, seed=9, level=5)
    x3 = oracle.prolong_disc(parent, xc, c, seed=10, level=4)
    assert not np.array_equal(x, x2) and not np.array_equal(x, x3)
    assert np.array_equal(x, oracle.prolong_disc(parent, xc, c, seed=9, level=4))


def test_init_box_range():
    x = oracle.init_box(500, 2, 7.5, seed=4, level=6)
    assert x.min() >= 0.0 and x.max() < 7.5
    U = oracle.uniform24(oracle.key_vertex(4, oracle.TAG_INIT, 6, 17, 2, 1))
    assert x[17, 1] == 7.5 * U


def test_coarse_sset_distances():
    """P:247-248 / Q7: d = c_u^(1/dim) + c_v^(1/dim), w = d^-2."""
    lvl = oracle.Level(n=2, row_ptr=np.array([0, 1, 2]), col=np.array([1, 0], dtype=np.int32),
                       omega=np.array([1, 1]), c=np.array([4, 9]), parent=None, rounds=0)
    cs = oracle.coarse_sset(lvl, 2)
    np.testing.assert_allclose(cs.d, [5.0, 5.0])
    np.testing.assert_allclose(cs.w, [0.04, 0.04])
    lvl3 = oracle.Level(n=2, row_ptr=np.array([0, 1, 2]), col=np.array([1, 0], dtype=np.int32),
                        omega=np.array([1, 1]), c=np.array([8, 27]), parent=None, rounds=0)
    np.testing.assert_allclose(oracle.coarse_sset(lvl3, 3).d, [5.0, 5.0], rtol=1e-15)


def test_layout_h0_equals_repeated_sweeps():
    w = configs.make("cfg1_grid12")
    x0 = w.x0.astype(np.float64)
    x, e, nl = oracle.layout(w.graph, w.S, 2, w.alpha, w.q, 0, [5], w.seed, x_init=x0)
    y = x0
    for _ in range(5):
        y = oracle.sweep_exact(w.S, y, w.alpha, w.q)
    np.testing.assert_array_equal(x, y)
    np.testing.assert_allclose(e, oracle.energy(w.S, y, w.alpha, w.q), rtol=0)
    assert nl == 1


def test_layout_multilevel_small_runs():
    w = configs.make("cfg3_mesh32")
    x, e, nl = oracle.layout(w.graph, w.S, 2, w.alpha, w.q, 2, [4], w.seed, n_stop=100)
    assert nl >= 3 and np.all(np.isfinite(x)) and np.isfinite(e[2])
    # the finest-level result is a pure function of the seed
    x2, e2, _ = oracle.layout(w.graph, w.S, 2, w.alpha, w.q, 2, [4], w.seed, n_stop=100)
    np.testing.assert_array_equal(x, x2)


# ---------------------------------------------------------------- SCLaP (f2, reading R6)
@pytest.mark.parametrize("name", ["cfg3_mesh64", "cfg5_grid16", "cfg4_cl20000"])
def test_sclap_hierarchy_invariants(name):
    """Cluster weights respect U = max(max c, min(2^h, n/f)); weights conserved;
    contraction = Pm^T A Pm; coarse ids rank the distinct labels."""
    w = configs.make(name)
    lv = oracle.build_hierarchy(w.graph, seed=w.seed, n_stop=100, sclap=True)
    assert len(lv) >= 3
    f = 20.0
    for l in range(len(lv) - 1):
        fine, coarse = lv[l], lv[l + 1]
        P = fine.parent
        k = coarse.n
        np.testing.assert_array_equal(np.bincount(P, weights=fine.c, minlength=k).astype(np.int64), coarse.c)
        W = min(2.0 ** (l + 1), w.n / f)
        U = max(int(fine.c.max()), int(W))
        assert coarse.c.max() <= U, (l, coarse.c.max(), U)
        n = fine.n
        A = sp.csr_matrix((fine.omega.astype(np.float64), fine.col, fine.row_ptr), shape=(n, n))
        Pm = sp.csr_matrix((np.ones(n), (np.arange(n), P)), shape=(n, k))
        C = (Pm.T @ A @ Pm).tocsr()
        C.setdiag(0)
        C.eliminate_zeros()
        C.sort_indices()
        np.testing.assert_array_equal(C.indptr, coarse.row_ptr)
        np.testing.assert_array_equal(C.indices, coarse.col)
        if 10 * coarse.n > 9 * fine.n:
            f *= 0.7


def test_sclap_triangle_single_cluster():
    """Triangle, U = 3: node 1 joins label 0; node 2 joins 0 or 1 (hash tie);
    the next round moves everything into label 0 (re-derived for R6)."""
    g = graphs.from_edges(3, np.array([0, 0, 1]), np.array([1, 2, 2]))
    lab = oracle.sclap_labels(g, U=3, rounds=3, seed=42, level=0)
    assert lab.tolist() == [0, 0, 0]


def test_sclap_size_bound_blocks_merge():
    """Path 0-1-2-3 with U = 2: every accepted cluster weighs <= 2."""
    g = H.path(4)
    lab = oracle.sclap_labels(g, U=2, rounds=5, seed=1, level=0)
    assert np.bincount(lab).max() <= 2
    assert lab[1] == 0  # node 1 moves to the smaller label 0 in round 0


# ---------------------------------------------------------------- SCLaP, the paper's sequential rule (R6s)
def _two_cliques(k):
    u, v = [], []
    for base in (0, k):
        for a in range(k):
            for b in range(a + 1, k):
                u.append(base + a)
                v.append(base + b)
    u.append(k - 1)
    v.append(k)  # the bridge
    return graphs.from_edges(2 * k, np.array(u), np.array(v))


def test_sclap_seq_two_cliques():
    """"nodes in a dense cluster usually agree on a common label":
    two K6 joined by one edge, U = 6 (a clique fits exactly), one label per
    clique whatever the random order (several seeds)."""
    g = _two_cliques(6)
    for seed in range(8):
        lab = oracle.sclap_labels(g, U=6, rounds=5, seed=seed, level=0, seq=True)
        assert len(set(lab[:6].tolist())) == 1 and len(set(lab[6:].tolist())) == 1, (seed, lab)
        assert lab[0] != lab[6]


def test_sclap_seq_bound_and_conservation():
    """every cluster weighs <= U after every label change; the
    weights of the nodes are conserved (labels partition the nodes)."""
    w = configs.make("cfg3_mesh32")
    rng = np.random.default_rng(3)
    c = rng.integers(1, 4, w.n).astype(np.int64)
    for U in (3, 5, 9):
        lab = oracle.sclap_labels(w.graph, U=U, rounds=4, seed=7, level=1, c=c, seq=True)
        cw = np.bincount(lab, weights=c, minlength=w.n)
        assert cw.max() <= U and cw.sum() == c.sum()


def test_sclap_seq_no_room_no_move():
    """U = max c: no cluster can take another node, so no label changes."""
    w = configs.make("cfg3_mesh32")
    lab = oracle.sclap_labels(w.graph, U=1, rounds=3, seed=1, level=0, seq=True)
    assert np.array_equal(lab, np.arange(w.n))


def test_sclap_seq_predominant_label_at_the_end():
    """A fixed point of the rule: after a round without moves, no node has an
    admissible label (not overloaded after the change) with a strictly larger
    edge weight than its own cluster's."""
    w = configs.make("cfg3_mesh32")
    U = 4
    lab = oracle.sclap_labels(w.graph, U=U, rounds=200, seed=5, level=0, seq=True)
    cw = np.bincount(lab, minlength=w.n)
    rp, col = w.graph.row_ptr, w.graph.col
    for v in range(w.n):
        sc = {}
        for j in col[rp[v]:rp[v + 1]]:
            sc[lab[j]] = sc.get(lab[j], 0) + 1
        own = sc.get(lab[v], 0)
        for L, s in sc.items():
            if L != lab[v] and cw[L] + 1 <= U:
                assert s <= own, (v, L, s, own)


def test_sclap_seq_immediate_updates_differ_from_synchronous():
    """The sequential rule sees moves made earlier in the same round (P:207
    "visits all nodes ... and assigns"), the synchronous reading R6 does not:
    on a long path with a large U one sequential round already forms clusters
    of more than two nodes, which one R6 round cannot (each node moves at most
    once, to a label that was a singleton at the start of the round)."""
    g = H.path(200)
    seq = oracle.sclap_labels(g, U=50, rounds=1, seed=3, level=0, seq=True)
    syn = oracle.sclap_labels(g, U=50, rounds=1, seed=3, level=0)
    assert np.bincount(seq).max() > 2
    assert np.bincount(syn).max() <= 2


@pytest.mark.parametrize("name", ["cfg3_mesh64", "cfg5_grid16", "cfg4_cl20000"])
def test_sclap_seq_hierarchy_invariants(name):
    """The paper's SCLaP hierarchy (R6s): U bound per level, conservation."""
    w = configs.make(name)
    lv = oracle.build_hierarchy(w.graph, seed=w.seed, n_stop=100, sclap=True, sclap_seq=True)
    assert len(lv) >= 3
    for l in range(len(lv) - 1):
        fine, coarse = lv[l], lv[l + 1]
        np.testing.assert_array_equal(np.bincount(fine.parent, weights=fine.c, minlength=coarse.n).astype(np.int64),
                                      coarse.c)
        assert coarse.c.max() <= max(int(fine.c.max()), int(2.0 ** (l + 1)))


def test_sclap_synchronous_reading_quality_vs_paper_rule():
    """The synchronous reading R6 (what the GPU runs) against the paper's
    sequential rule on the same graphs: both coarsen geometrically to the
    stop size, R6 within a few levels of the sequential hierarchy, and the
    paper's full optimizer (SCLaP + disc prolongation + alpha schedule, h = 2)
    reaches a final maxent-stress energy of the same quality (geometric mean
    ratio within [2/3, 3/2] over the instances)."""
    ratios = []
    for name in ("cfg3_mesh64", "cfg5_grid12", "cfg3_mesh128"):
        w = configs.make(name)
        lr = oracle.build_hierarchy(w.graph, seed=w.seed, n_stop=100, sclap=True)
        ls = oracle.build_hierarchy(w.graph, seed=w.seed, n_stop=100, sclap=True, sclap_seq=True)
        assert lr[-1].n <= 100 and ls[-1].n <= 100
        assert abs(len(lr) - len(ls)) <= 3, ([l.n for l in lr], [l.n for l in ls])
        for fine, coarse in zip(lr[:-1], lr[1:]):
            assert coarse.n <= 0.9 * fine.n
        sched = oracle.paper_schedule(max_final_iters=30)
        e = [oracle.layout_schedule(w.graph, w.S, w.dim, w.q, 2, sched, w.seed, n_stop=100, sclap=True, disc=True,
                                    sclap_seq=s)[1][2] for s in (False, True)]
        assert e[0] > 0 and e[1] > 0
        ratios.append(e[0] / e[1])
    g = float(np.exp(np.mean(np.log(ratios))))
    assert 2.0 / 3.0 <= g <= 1.5, ratios
