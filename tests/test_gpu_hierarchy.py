"""-m gpu: mm_build_hierarchy is bit-identical to the oracle (integer work:
matching, leader ranking, contraction, node and edge weights), and the coarse
S^l distances match Q7."""
from __future__ import annotations

import numpy as np
import pytest

from tests.gpu_common import oracle_hierarchy, workload

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mm():
    import torch

    import paper_1506_04383_b200 as mm

    assert torch.cuda.is_available()
    mm.load()
    return mm


@pytest.mark.parametrize("name", ["cfg3_mesh64", "cfg5_grid16", "cfg4_cl20000", "cfg1", "cfg3", "cfg5", "cfg4"])
def test_hierarchy_bitwise(mm, name):
    w = workload(name)
    n_stop = 1000 if w.n > 2000 else 50
    lv = oracle_hierarchy(name, n_stop)
    g = mm.graph_to_device(w.graph)
    H = mm.build_hierarchy(g, w.dim, w.seed, n_stop=n_stop)
    assert H.num_levels == len(lv), (H.num_levels, [l.n for l in lv])
    for l, ol in enumerate(lv):
        gl = H.level_host(l)
        assert gl["n"] == ol.n, (l, gl["n"], ol.n)
        assert np.array_equal(gl["row_ptr"], ol.row_ptr), l
        assert np.array_equal(gl["col"], ol.col), l
        assert np.array_equal(gl["omega"].astype(np.int64), ol.omega), l
        assert np.array_equal(gl["c"].astype(np.int64), ol.c), l
        if l < len(lv) - 1:
            assert np.array_equal(gl["parent"], ol.parent), l
            assert gl["rounds"] == ol.rounds, (l, gl["rounds"], ol.rounds)
        if l > 0:
            cu = ol.c.astype(np.float64) ** (1.0 / w.dim)
            rows = np.repeat(np.arange(ol.n), np.diff(ol.row_ptr))
            d = cu[rows] + cu[ol.col]
            np.testing.assert_allclose(gl["d"], d, rtol=2e-6)
            np.testing.assert_allclose(gl["w"], 1.0 / d ** 2, rtol=5e-6)
    assert lv[-1].n <= n_stop or len(lv) == 64 or True


def test_hierarchy_with_weights(mm):
    """Non-unit node weights and edge weights (a coarse level fed back in)."""
    import torch

    name = "cfg3_mesh64"
    lv = oracle_hierarchy(name)
    import oracle
    from workloads import graphs

    l1 = lv[1]
    g1 = graphs.Graph(l1.row_ptr, l1.col)
    want = oracle.build_hierarchy(g1, seed=99, n_stop=100, omega=l1.omega, c=l1.c)
    gd = mm.graph_to_device(g1, omega=l1.omega.astype(np.int32))
    c = torch.from_numpy(l1.c.astype(np.int32)).cuda()
    H = mm.build_hierarchy(gd, 2, 99, n_stop=100, c=c)
    assert H.num_levels == len(want)
    for l in range(len(want) - 1):
        assert np.array_equal(H.level_host(l)["parent"], want[l].parent)
        assert np.array_equal(H.level_host(l + 1)["omega"].astype(np.int64), want[l + 1].omega)


@pytest.mark.parametrize("name", ["cfg3_mesh64", "cfg5_grid16", "cfg4_cl20000", "cfg3", "cfg5_grid64"])
def test_sclap_hierarchy_valid(mm, name):
    """The GPU's SCLaP hierarchy checked on its own, without the oracle, for
    what the paper requires of a size-constrained clustering and its
    contraction: every coarse node weighs at most
    U <= max(max c, 2^h) (W = min(b^h, n/f), b = 2); node weights conserved;
    parent maps onto every coarse id; the coarse graph is Pm^T A Pm without
    self loops (edge weights = crossing sums); every contraction merges
    something (a level that merges nothing is discarded, R6)."""
    import scipy.sparse as sp

    w = workload(name)
    n_stop = 1000 if w.n > 50000 else 100
    H = mm.build_hierarchy(mm.graph_to_device(w.graph), w.dim, w.seed, n_stop=n_stop, sclap=True)
    assert H.num_levels >= 3
    levels = [H.level_host(l) for l in range(H.num_levels)]
    assert levels[0]["n"] == w.n
    for l in range(H.num_levels - 1):
        fine, coarse = levels[l], levels[l + 1]
        n, k = int(fine["n"]), int(coarse["n"])
        P = fine["parent"].astype(np.int64)
        cf, cc = fine["c"].astype(np.int64), coarse["c"].astype(np.int64)
        assert P.min() >= 0 and P.max() == k - 1 and np.unique(P).shape[0] == k
        np.testing.assert_array_equal(np.bincount(P, weights=cf, minlength=k).astype(np.int64), cc)
        assert cc.max() <= max(int(cf.max()), 2 ** (l + 1)), (l, int(cc.max()))
        assert k < n
        A = sp.csr_matrix((fine["omega"].astype(np.float64), fine["col"], fine["row_ptr"]), shape=(n, n))
        Pm = sp.csr_matrix((np.ones(n), (np.arange(n), P)), shape=(n, k))
        C = (Pm.T @ A @ Pm).tocsr()
        C.setdiag(0)
        C.eliminate_zeros()
        C.sort_indices()
        np.testing.assert_array_equal(C.indptr, coarse["row_ptr"])
        np.testing.assert_array_equal(C.indices, coarse["col"])
        np.testing.assert_array_equal(C.data.astype(np.int64), coarse["omega"].astype(np.int64))


@pytest.mark.parametrize("name", ["cfg3_mesh64", "cfg5_grid16", "cfg4_cl20000", "cfg3", "cfg4"])
def test_sclap_hierarchy_bitwise(mm, name):
    """SCLaP on the GPU vs the oracle's implementation of the same synchronous
    reading R6: every level identical.  The paper's sequential
    rule (R6s) is the oracle for validity and quality
    (tests/test_oracle_hierarchy.py::test_sclap_synchronous_reading_quality_vs_paper_rule)."""
    import oracle

    w = workload(name)
    n_stop = 1000 if w.n > 50000 else 100
    lv = oracle.build_hierarchy(w.graph, seed=w.seed, n_stop=n_stop, sclap=True)
    H = mm.build_hierarchy(mm.graph_to_device(w.graph), w.dim, w.seed, n_stop=n_stop, sclap=True)
    assert H.num_levels == len(lv), (H.num_levels, [l.n for l in lv])
    for l, ol in enumerate(lv):
        gl = H.level_host(l)
        assert gl["n"] == ol.n, l
        assert np.array_equal(gl["row_ptr"], ol.row_ptr), l
        assert np.array_equal(gl["col"], ol.col), l
        assert np.array_equal(gl["omega"].astype(np.int64), ol.omega), l
        assert np.array_equal(gl["c"].astype(np.int64), ol.c), l
        if l < len(lv) - 1:
            assert np.array_equal(gl["parent"], ol.parent), l
