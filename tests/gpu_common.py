"""Shared helpers for the -m gpu parity tests (oracle vs CUDA path on the same
seeded inputs).  Tolerance (BASELINE.json north_star): after one sweep from an
identical state, max |x_gpu - x_oracle| <= 1e-4 x the diagonal of the oracle
output's bounding box; full runs: final energy within 1e-3 relative."""
from __future__ import annotations

import functools

import numpy as np

SWEEP_TOL = 1e-4
ENERGY_TOL = 1e-3


@functools.lru_cache(maxsize=None)
def workload(name: str):
    from workloads import configs

    return configs.make(name)


@functools.lru_cache(maxsize=None)
def oracle_hierarchy(name: str, n_stop: int = 1000):
    import oracle

    w = workload(name)
    return oracle.build_hierarchy(w.graph, seed=w.seed, n_stop=n_stop)


def bbox_diameter(x: np.ndarray) -> float:
    return float(np.linalg.norm(x.max(axis=0) - x.min(axis=0)))


def assert_sweep_parity(got: np.ndarray, want: np.ndarray, what: str, tol: float = SWEEP_TOL) -> float:
    assert got.shape == want.shape, (got.shape, want.shape)
    assert np.all(np.isfinite(got)), f"{what}: non-finite GPU output"
    diam = bbox_diameter(want)
    err = float(np.abs(got - want).max())
    assert err <= tol * diam, f"{what}: max |gpu - oracle| = {err:.3e} > {tol} x diameter {diam:.3e}"
    return err / diam


def sample_rows(n: int, count: int, seed: int, extra=()) -> np.ndarray:
    rng = np.random.default_rng(seed)
    rows = rng.choice(n, size=min(count, n), replace=False)
    rows = np.unique(np.concatenate([rows, np.asarray(extra, dtype=np.int64), [0, n - 1]]))
    return rows.astype(np.int32)


def rel_diff(a: float, b: float) -> float:
    return abs(a - b) / max(abs(b), 1e-300)


def assert_energy_or_chaos(e_gpu: float, e_oracle: float, control, what: str, factor: float = 2.0,
                           perturbation: float = 1e-6):
    """Full-run parity (Q20): |E_gpu - E_oracle| <= 1e-3 |E_oracle|,
    or, when the trajectory is chaotic, within `factor` x the divergence of the
    oracle from itself under a +-`perturbation` relative change of alpha
    (control(s) -> oracle energy).  1e-6 is the scale of FP32 rounding
    accumulated over a sweep (a few ulp of 6e-8 per operation chain)."""
    rel = rel_diff(e_gpu, e_oracle)
    if rel <= ENERGY_TOL:
        return
    ctrl = max(rel_diff(control(s), e_oracle) for s in (perturbation, -perturbation))
    assert rel <= factor * ctrl, (what, rel, ctrl)
    print(f"{what}: |E_gpu - E_oracle| / |E| = {rel:.2e} > {ENERGY_TOL}; chaos control {ctrl:.2e}")
