"""Shared helpers for the -m gpu parity tests (oracle vs CUDA path on the same
seeded inputs).  Tolerance (BASELINE.json north_star): after one sweep from an
identical state, max |x_gpu - x_oracle| <= 1e-4 x the diagonal of the oracle
output's bounding box; full runs: final energy within 1e-3 relative."""
from __future__ import annotations

import functools
import json
import os

import numpy as np

SWEEP_TOL = 1e-4
ENERGY_TOL = 1e-3
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


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


PARITY_LOG = os.environ.get("MM_PARITY_LOG", os.path.join(ROOT, "gpurun_out", "fullrun_parity.jsonl"))


def log_parity(record: dict) -> None:
    """Appends one JSON line per full-run case to PARITY_LOG (every case, pass
    or fail), so the relative errors of a -m gpu run are on record."""
    os.makedirs(os.path.dirname(PARITY_LOG), exist_ok=True)
    with open(PARITY_LOG, "a") as f:
        f.write(json.dumps(record) + "\n")


def assert_energy(e_gpu: float, e_oracle: float, what: str, **extra) -> float:
    """Full-run parity, BASELINE.json north_star: |E_gpu - E_oracle| <=
    1e-3 |E_oracle| (final energy Eq.(1)).  No escape branch: the
    case is logged and then asserted."""
    rel = rel_diff(e_gpu, e_oracle)
    log_parity({"case": what, "E_gpu": e_gpu, "E_oracle": e_oracle, "rel": rel, "bar": ENERGY_TOL,
                "pass": rel <= ENERGY_TOL, **extra})
    assert rel <= ENERGY_TOL, f"{what}: |E_gpu - E_oracle| / |E_oracle| = {rel:.3e} > {ENERGY_TOL}"
    return rel
