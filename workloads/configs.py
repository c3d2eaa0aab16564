"""The five BASELINE.json configs (plus scaled-down same-generator variants
for oracle-sized tests).  Seeds: graph seed = 1000 + K for config K (SURVEY
§8(d)); the initial-coordinate stream uses a separate seed.

`make(name)` returns a Workload with the graph, the S set, the scalar
parameters and (for single-level exact configs) the FP32 initial
coordinates, which are generated here once and passed identically to both
the oracle and the CUDA path.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import graphs, sset


@dataclass
class Workload:
    name: str
    graph: graphs.Graph
    S: sset.SSet
    dim: int
    alpha: float
    q: float
    h: int                   # 0: exact single level; >0: multilevel, h-level approximation
    sweeps: int              # sweeps per level
    seed: int                # method seed (matching tie-break, init, jitter)
    x0: Optional[np.ndarray] = None   # float32 [n, dim] for exact single-level configs
    meta: dict = field(default_factory=dict)

    @property
    def n(self) -> int:
        return self.graph.n


def init_coords(n: int, dim: int, seed: int) -> np.ndarray:
    """x0 ~ U[0,1)^dim, float32, from its own seeded stream."""
    rng = np.random.default_rng(seed)
    return rng.random((n, dim), dtype=np.float32)


def random_state(n: int, dim: int, seed: int, scale: float = 1.0) -> np.ndarray:
    """A seeded float32 layout state for one-sweep parity cases."""
    rng = np.random.default_rng(seed)
    return (rng.random((n, dim), dtype=np.float32) * np.float32(scale)).astype(np.float32)


def _cfg1(scale: int = 32) -> Workload:
    g = graphs.grid2d(scale, scale)
    S = sset.edges_sset(g)
    return Workload("cfg1" if scale == 32 else f"cfg1_grid{scale}", g, S, dim=2, alpha=0.1, q=0.0,
                    h=0, sweeps=50, seed=1001, x0=init_coords(g.n, 2, 2001))


def _cfg2(n: int = 65536) -> Workload:
    g, pts = graphs.rgg(n, seed=1002)
    S = sset.hop2_sset(g)
    return Workload("cfg2" if n == 65536 else f"cfg2_rgg{n}", g, S, dim=2, alpha=0.01, q=0.0,
                    h=0, sweeps=20, seed=1002, x0=init_coords(g.n, 2, 2002))


def _cfg3(side: int = 512) -> Workload:
    g = graphs.trimesh(side, seed=1003)
    S = sset.hop2_sset(g)
    return Workload("cfg3" if side == 512 else f"cfg3_mesh{side}", g, S, dim=2, alpha=0.01,
                    q=0.0, h=2, sweeps=30, seed=1003)


def _cfg4(n: int = 1 << 20) -> Workload:
    g = graphs.chung_lu(n, seed=1004)
    S = sset.capped_sset(g, 64)
    return Workload("cfg4" if n == (1 << 20) else f"cfg4_cl{n}", g, S, dim=2, alpha=0.005,
                    q=0.0, h=2, sweeps=20, seed=1004)


def _cfg5(side: int = 128) -> Workload:
    g = graphs.grid3d(side, side, side)
    S = sset.edges_sset(g)
    return Workload("cfg5" if side == 128 else f"cfg5_grid{side}", g, S, dim=3, alpha=0.01,
                    q=0.8, h=2, sweeps=15, seed=1005)


def make(name: str) -> Workload:
    """Full configs: cfg1..cfg5.  Scaled variants: 'cfg1_grid<k>', 'cfg2_rgg<n>',
    'cfg3_mesh<side>', 'cfg4_cl<n>', 'cfg5_grid<side>'."""
    if name == "cfg1":
        return _cfg1()
    if name == "cfg2":
        return _cfg2()
    if name == "cfg3":
        return _cfg3()
    if name == "cfg4":
        return _cfg4()
    if name == "cfg5":
        return _cfg5()
    if name.startswith("cfg1_grid"):
        return _cfg1(int(name[len("cfg1_grid"):]))
    if name.startswith("cfg2_rgg"):
        return _cfg2(int(name[len("cfg2_rgg"):]))
    if name.startswith("cfg3_mesh"):
        return _cfg3(int(name[len("cfg3_mesh"):]))
    if name.startswith("cfg4_cl"):
        return _cfg4(int(name[len("cfg4_cl"):]))
    if name.startswith("cfg5_grid"):
        return _cfg5(int(name[len("cfg5_grid"):]))
    raise KeyError(name)
