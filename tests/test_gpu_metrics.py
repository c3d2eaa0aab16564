"""-m gpu: mm_full_stress against the oracle's
BFS-from-every-vertex evaluation on the same FP32 layouts."""
from __future__ import annotations

import numpy as np
import pytest

import oracle
from tests import helpers as H
from tests.gpu_common import workload
from workloads import configs

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mm():
    import torch

    import paper_1506_04383_b200 as mm

    assert torch.cuda.is_available()
    mm.load()
    return mm


@pytest.mark.parametrize("name,dim", [("cfg1", 2), ("cfg2_rgg4096", 2), ("cfg5_grid12", 3), ("cfg4_cl20000", 2)])
def test_full_stress_parity(mm, name, dim):
    w = workload(name)
    x = (w.x0 if w.x0 is not None else configs.random_state(w.n, dim, seed=5, scale=w.n ** (1 / dim)))
    got = mm.full_stress(mm.graph_to_device(w.graph), mm.coords_to_device(x))
    want = oracle.full_stress(w.graph, x.astype(np.float64))
    assert got[3] == want[3] == w.n * (w.n - 1) // 2
    np.testing.assert_allclose(got[:3], want[:3], rtol=1e-9)


def test_full_stress_worked_examples(mm):
    F, s, Fs, P = mm.full_stress(mm.graph_to_device(H.path(3)),
                                 mm.coords_to_device(np.array([[0.0, 0], [1, 0], [2, 0]], np.float32)))
    assert (F, s, P) == (0.0, 1.0, 3)
    F, s, Fs, P = mm.full_stress(mm.graph_to_device(H.path(2)),
                                 mm.coords_to_device(np.array([[0.0, 0], [3, 0]], np.float32)))
    assert F == 4.0 and abs(s - 1 / 3) < 1e-15 and abs(Fs) < 1e-15
