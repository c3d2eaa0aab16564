"""-m gpu: element-wise parity of the prolongation kernels (k_prolong,
k_prolong_disc through mm_prolong) with the oracle's or_prolong /
or_prolong_disc.

Q15 (BASELINE.json configs[2]): x_u = x_P(u) + 1e-3 (2U - 1) per component.
Disc (R7): angle 2 pi U0, distance c(P(u))^(1/dim) U1.
The counter RNG draws are compared exactly (recovered from the output with
the coarse coordinates at 0); coordinates to FP32 rounding.
"""
from __future__ import annotations

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mm():
    import torch

    import paper_1506_04383_b200 as mm

    assert torch.cuda.is_available()
    mm.load()
    return mm


def _case(dim, n=50_000, nc=777, seed=3):
    rng = np.random.default_rng(seed)
    parent = rng.integers(0, nc, n).astype(np.int32)
    xc = (rng.normal(size=(nc, dim)) * 300.0).astype(np.float32)
    c = rng.integers(1, 60, nc).astype(np.int32)
    return parent, xc, c


def _dev(mm, a):
    import torch

    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


@pytest.mark.parametrize("dim", [2, 3])
def test_prolong_jitter_matches_oracle(mm, dim):
    parent, xc, _ = _case(dim)
    got = mm.coords_from_device(mm.prolong(_dev(mm, parent), mm.coords_to_device(xc), seed=1003, level=2), dim)
    want = oracle.prolong(parent, xc.astype(np.float64), seed=1003, level=2)
    # FP32 result of xc + 1e-3 (2U - 1): within one rounding of |x| plus the 1e-3 step
    tol = 2.0 * np.finfo(np.float32).eps * (np.abs(want) + 1e-3)
    assert np.all(np.abs(got - want) <= tol), float(np.max(np.abs(got - want) / tol))


@pytest.mark.parametrize("dim", [2, 3])
def test_prolong_jitter_rng_draws_exact(mm, dim):
    """xc = 0: the output is 1e-3f (2U - 1) with U = m / 2^24; recover m and
    compare it with the oracle's draw bit for bit (same keys, same bits)."""
    n = 20_000
    parent = np.zeros(n, dtype=np.int32)
    xc = np.zeros((1, dim), dtype=np.float32)
    got = mm.coords_from_device(mm.prolong(_dev(mm, parent), mm.coords_to_device(xc), seed=77, level=5), dim)
    m_gpu = np.rint((got.astype(np.float64) / np.float64(np.float32(1e-3)) + 1.0) * 0.5 * 2 ** 24).astype(np.int64)
    want = oracle.prolong(parent, xc.astype(np.float64), seed=77, level=5)
    m_or = np.rint((want / 1e-3 + 1.0) * 0.5 * 2 ** 24).astype(np.int64)
    assert np.array_equal(m_gpu, m_or)
    # and the oracle's draws are the pinned RNG's (tests/golden/splitmix64.txt pins mix64)
    U = oracle.uniform24(oracle.key_vertex(77, oracle.TAG_JITTER, 5, 123, dim, dim - 1))
    assert m_or[123, dim - 1] == int(U * 2 ** 24)


@pytest.mark.parametrize("dim", [2, 3])
def test_prolong_disc_matches_oracle(mm, dim):
    parent, xc, c = _case(dim, seed=4)
    got = mm.coords_from_device(mm.prolong(_dev(mm, parent), mm.coords_to_device(xc), seed=1005, level=1,
                                           c_coarse=_dev(mm, c)), dim)
    want = oracle.prolong_disc(parent, xc.astype(np.float64), c.astype(np.int64), seed=1005, level=1)
    r = c[parent].astype(np.float64) ** (1.0 / dim)
    # FP32: |x| rounding plus sincos of a 2 pi U0 argument rounded to FP32 (~1e-6 r)
    tol = 4.0 * np.finfo(np.float32).eps * np.abs(want) + 2e-6 * r[:, None]
    assert np.all(np.abs(got - want) <= tol), float(np.max(np.abs(got - want) / tol))
    # every vertex inside its parent's disc / ball
    dist = np.linalg.norm(got.astype(np.float64) - xc[parent].astype(np.float64), axis=1)
    assert np.all(dist <= r * (1 + 1e-5) + 1e-4)


def test_prolong_empty_and_bad_args(mm):
    import torch

    xc = mm.coords_to_device(np.zeros((4, 2), dtype=np.float32))
    out = mm.prolong(torch.zeros(0, dtype=torch.int32, device="cuda"), xc, seed=1, level=0)
    assert out.shape[0] == 0
    with pytest.raises(mm.MMError):
        mm.prolong(torch.zeros(4, dtype=torch.int32, device="cuda"), xc, seed=1, level=0, out=xc)
