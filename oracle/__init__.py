"""MulMent ORACLE — TEST INFRASTRUCTURE ONLY.

A plain FP64 CPU implementation of the maxent-stress hot path, written from
PAPER.md (arXiv 1506.04383) in C (oracle/*.c) and exposed here through ctypes
+ numpy.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs may import this package.  It shares no code with the
CUDA path (paper_1506_04383_b200/) and never imports it.

Parity status per function:
  sweep_exact      pinned (P1 2-path orbit, P2 3-path fixed point, P3 ring closed
                   form, P4 SPEC worked example, P5 conservation, P6 equivariance,
                   P7 descent, P10 SMACOF/scipy special case)
  sweep_approx     pinned (P9 identity map / single cluster / hand instance)
  energy           pinned (P4 worked example, P8 brute-force double loop)
  build_hierarchy  pinned (P11 invariants, brute-force contraction, hand instances)
  centroids        pinned (P12 independent recomputation)
  prolong/init     pinned (P13 bounds; RNG pinned to SplitMix64's published vector)
  prolong_disc     pinned (radius <= c^(1/dim); distance / r uniform on [0, 1] and
                   angle / direction uniform, the laws P:242 states; RNG keys)
  layout           parity unpinned by the paper for full multilevel trajectories
                   (Q20); its pieces are pinned individually.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass
from typing import List, Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_SRCS = ["rng.c", "sweep.c", "energy.c", "hierarchy.c", "layout.c", "schedule.c", "fullstress.c", "sclap.c"]

OR_EINVAL, OR_ERHO, OR_ECOINC, OR_ENOMEM = -1, -2, -3, -4
TAG_INIT, TAG_JITTER, TAG_MATCH = 0x494E4954, 0x4A495454, 0x4D415443


class OracleError(RuntimeError):
    def __init__(self, code: int, what: str):
        names = {OR_EINVAL: "EINVAL", OR_ERHO: "ERHO (rho_i <= 0)",
                 OR_ECOINC: "ECOINC (coincident non-S pair)", OR_ENOMEM: "ENOMEM"}
        super().__init__(f"{what}: {names.get(code, code)}")
        self.code = code


def build(force: bool = False) -> str:
    srcs = [os.path.join(_HERE, s) for s in _SRCS] + [os.path.join(_HERE, "mm_oracle.h")]
    if (not force and os.path.exists(_LIB_PATH)
            and all(os.path.getmtime(_LIB_PATH) >= os.path.getmtime(s) for s in srcs)):
        return _LIB_PATH
    cmd = ["gcc", "-O2", "-std=c11", "-fopenmp", "-fno-fast-math", "-ffp-contract=off",
           "-shared", "-fPIC", "-o", _LIB_PATH] + [os.path.join(_HERE, s) for s in _SRCS] + ["-lm"]
    subprocess.check_call(cmd)
    return _LIB_PATH


class Schedule(ctypes.Structure):
    """or_schedule: the paper's defaults; max_final_iters is a safety cap."""
    _fields_ = [("alpha0", ctypes.c_double), ("alpha_min", ctypes.c_double), ("factor", ctypes.c_double),
                ("eps", ctypes.c_double), ("a", ctypes.c_int32), ("max_final_iters", ctypes.c_int32)]


def paper_schedule(**kw) -> Schedule:
    v = dict(alpha0=1.0, alpha_min=0.008, factor=0.3, eps=1e-4, a=2, max_final_iters=200)
    v.update(kw)
    return Schedule(**v)


_lib = None
_i64p = ctypes.POINTER(ctypes.c_int64)
_i32p = ctypes.POINTER(ctypes.c_int32)
_f64p = ctypes.POINTER(ctypes.c_double)


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    build()
    L = ctypes.CDLL(_LIB_PATH)
    c_i32, c_i64, c_int, c_dbl, c_u64 = ctypes.c_int32, ctypes.c_int64, ctypes.c_int, ctypes.c_double, ctypes.c_uint64
    L.or_mix64.argtypes = [c_u64]; L.or_mix64.restype = c_u64
    L.or_uniform24.argtypes = [c_u64]; L.or_uniform24.restype = c_dbl
    L.or_key_vertex.argtypes = [c_u64, c_u64, c_u64, c_u64, c_int, c_int]; L.or_key_vertex.restype = c_u64
    L.or_sweep_exact.argtypes = [c_i32, c_int, _i64p, _i32p, _f64p, _f64p, _f64p, c_dbl, c_dbl,
                                 _i32p, c_i32, _f64p, c_int]
    L.or_centroids.argtypes = [c_i32, c_int, _f64p, _i32p, c_i32, _f64p, _i64p]
    L.or_sweep_approx.argtypes = [c_i32, c_int, _i64p, _i32p, _f64p, _f64p, _f64p, c_dbl, c_dbl,
                                  _i32p, _i32p, c_i32, _i32p, c_i32, _f64p, c_int]
    L.or_energy.argtypes = [c_i32, c_int, _i64p, _i32p, _f64p, _f64p, _f64p, c_dbl, c_dbl, _f64p, c_int]
    L.or_relative_change.argtypes = [c_i64, _f64p, _f64p]; L.or_relative_change.restype = c_dbl
    L.or_build_hierarchy.argtypes = [c_i32, _i64p, _i32p, _i64p, _i64p, c_u64, c_i32, c_i32, c_i32,
                                     ctypes.POINTER(ctypes.c_void_p)]
    L.or_hier_num_levels.argtypes = [ctypes.c_void_p]; L.or_hier_num_levels.restype = c_i32
    L.or_hier_level.argtypes = [ctypes.c_void_p, c_i32, _i32p, _i64p, ctypes.POINTER(_i64p),
                                ctypes.POINTER(_i32p), ctypes.POINTER(_i64p), ctypes.POINTER(_i64p),
                                ctypes.POINTER(_i32p), _i32p]
    L.or_hier_free.argtypes = [ctypes.c_void_p]; L.or_hier_free.restype = None
    L.or_coarse_sset.argtypes = [c_i32, c_i64, _i64p, _i32p, _i64p, c_int, _f64p, _f64p]
    L.or_init_box.argtypes = [c_i32, c_int, c_dbl, c_u64, c_i32, _f64p]
    L.or_prolong.argtypes = [c_i32, c_int, _i32p, _f64p, c_u64, c_i32, _f64p]
    L.or_prolong_disc.argtypes = [c_i32, c_int, _i32p, _f64p, _i64p, c_u64, c_i32, _f64p]
    L.or_layout.argtypes = [c_i32, c_int, _i64p, _i32p, _i64p, _i32p, _f64p, _f64p, c_dbl, c_dbl, c_int,
                            _i32p, c_i32, c_u64, c_i32, _f64p, _f64p, _f64p, _i32p, c_int]
    L.or_layout_schedule.argtypes = [c_i32, c_int, _i64p, _i32p, _i64p, _i32p, _f64p, _f64p, c_dbl, c_int,
                                     ctypes.POINTER(Schedule), c_u64, c_i32, c_int, _f64p, _f64p, _f64p, _i32p, _i32p,
                                     c_int]
    L.or_full_stress.argtypes = [c_i32, _i64p, _i32p, c_int, _f64p, _f64p, c_int]
    L.or_build_hierarchy_sclap.argtypes = [c_i32, _i64p, _i32p, _i64p, _i64p, c_u64, c_i32, c_i32, c_i32, c_dbl, c_dbl,
                                           ctypes.POINTER(ctypes.c_void_p)]
    L.or_sclap_labels.argtypes = [c_i32, _i64p, _i32p, _i64p, _i64p, c_i64, c_i32, c_u64, c_i32, _i32p]
    L.or_sclap_labels_seq.argtypes = [c_i32, _i64p, _i32p, _i64p, _i64p, c_i64, c_i32, c_u64, c_i32, _i32p]
    L.or_build_hierarchy_sclap_mode.argtypes = [c_i32, _i64p, _i32p, _i64p, _i64p, c_u64, c_i32, c_i32, c_i32, c_dbl,
                                                c_dbl, c_int, ctypes.POINTER(ctypes.c_void_p)]
    _lib = L
    return L


def _p(a: Optional[np.ndarray], t):
    if a is None:
        return ctypes.cast(None, ctypes.POINTER(t))
    return a.ctypes.data_as(ctypes.POINTER(t))


def _csr(S):
    rp = np.ascontiguousarray(S.row_ptr, dtype=np.int64)
    col = np.ascontiguousarray(S.col, dtype=np.int32)
    d = np.ascontiguousarray(S.d, dtype=np.float64)
    w = np.ascontiguousarray(S.w, dtype=np.float64)
    return rp, col, d, w


def _check(rc: int, what: str):
    if rc != 0:
        raise OracleError(rc, what)


def default_threads() -> int:
    return int(os.environ.get("ORACLE_THREADS", os.cpu_count() or 1))


# ------------------------------------------------------------------ RNG
def mix64(z: int) -> int:
    return int(lib().or_mix64(ctypes.c_uint64(z & 0xFFFFFFFFFFFFFFFF)))


def uniform24(key: int) -> float:
    return float(lib().or_uniform24(ctypes.c_uint64(key)))


def key_vertex(seed: int, tag: int, level: int, vertex: int, dim: int, comp: int) -> int:
    return int(lib().or_key_vertex(seed, tag, level, vertex, dim, comp))


# ------------------------------------------------------------------ sweeps
def sweep_exact(S, x: np.ndarray, alpha: float, q: float, rows: Optional[np.ndarray] = None,
                nthreads: Optional[int] = None) -> np.ndarray:
    """Eq.(2), one Jacobi sweep; returns rows' new coords (FP64)."""
    rp, col, d, w = _csr(S)
    x = np.ascontiguousarray(x, dtype=np.float64)
    n, dim = x.shape
    r = None if rows is None else np.ascontiguousarray(rows, dtype=np.int32)
    nr = n if r is None else r.shape[0]
    out = np.empty((nr, dim), dtype=np.float64)
    _check(lib().or_sweep_exact(n, dim, _p(rp, ctypes.c_int64), _p(col, ctypes.c_int32),
                                _p(d, ctypes.c_double), _p(w, ctypes.c_double), _p(x, ctypes.c_double),
                                alpha, q, _p(r, ctypes.c_int32), nr, _p(out, ctypes.c_double),
                                nthreads or default_threads()), "sweep_exact")
    return out


def centroids(x: np.ndarray, anc: np.ndarray, k: int):
    """(x'[k, dim], nu[k]) — P:274, Q10-Q12."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    anc = np.ascontiguousarray(anc, dtype=np.int32)
    n, dim = x.shape
    xc = np.empty((k, dim), dtype=np.float64)
    nu = np.empty(k, dtype=np.int64)
    _check(lib().or_centroids(n, dim, _p(x, ctypes.c_double), _p(anc, ctypes.c_int32), k,
                              _p(xc, ctypes.c_double), _p(nu, ctypes.c_int64)), "centroids")
    return xc, nu


def sweep_approx(S, x: np.ndarray, alpha: float, q: float, parent: np.ndarray, anc: np.ndarray,
                 k: int, rows: Optional[np.ndarray] = None, nthreads: Optional[int] = None) -> np.ndarray:
    """Eq.(3), one Jacobi sweep; returns rows' new coords (FP64)."""
    rp, col, d, w = _csr(S)
    x = np.ascontiguousarray(x, dtype=np.float64)
    n, dim = x.shape
    parent = np.ascontiguousarray(parent, dtype=np.int32)
    anc = np.ascontiguousarray(anc, dtype=np.int32)
    r = None if rows is None else np.ascontiguousarray(rows, dtype=np.int32)
    nr = n if r is None else r.shape[0]
    out = np.empty((nr, dim), dtype=np.float64)
    _check(lib().or_sweep_approx(n, dim, _p(rp, ctypes.c_int64), _p(col, ctypes.c_int32),
                                 _p(d, ctypes.c_double), _p(w, ctypes.c_double), _p(x, ctypes.c_double),
                                 alpha, q, _p(parent, ctypes.c_int32), _p(anc, ctypes.c_int32), k,
                                 _p(r, ctypes.c_int32), nr, _p(out, ctypes.c_double),
                                 nthreads or default_threads()), "sweep_approx")
    return out


def energy(S, x: np.ndarray, alpha: float, q: float, nthreads: Optional[int] = None,
           skip_coincident: bool = False):
    """Eq.(1) (Q3/Q4): returns (stress, entropy, total).
    A coincident non-S pair is an error, unless skip_coincident: then
    such pairs are left out of the entropy, as mm_layout's report does (Q6)."""
    rp, col, d, w = _csr(S)
    x = np.ascontiguousarray(x, dtype=np.float64)
    n, dim = x.shape
    out = np.zeros(3, dtype=np.float64)
    rc = lib().or_energy(n, dim, _p(rp, ctypes.c_int64), _p(col, ctypes.c_int32),
                         _p(d, ctypes.c_double), _p(w, ctypes.c_double), _p(x, ctypes.c_double),
                         alpha, q, _p(out, ctypes.c_double), nthreads or default_threads())
    if not (skip_coincident and rc == -3):
        _check(rc, "energy")
    return float(out[0]), float(out[1]), float(out[2])


def relative_change(x_old: np.ndarray, x_new: np.ndarray) -> float:
    a = np.ascontiguousarray(x_old, dtype=np.float64).ravel()
    b = np.ascontiguousarray(x_new, dtype=np.float64).ravel()
    return float(lib().or_relative_change(a.shape[0], _p(a, ctypes.c_double), _p(b, ctypes.c_double)))


# ------------------------------------------------------------------ hierarchy
@dataclass
class Level:
    n: int
    row_ptr: np.ndarray
    col: np.ndarray
    omega: np.ndarray
    c: np.ndarray
    parent: Optional[np.ndarray]
    rounds: int


def build_hierarchy(g, seed: int, n_stop: int = 1000, max_levels: int = 64, max_rounds: int = 64,
                    omega: Optional[np.ndarray] = None, c: Optional[np.ndarray] = None, sclap: bool = False,
                    lp_rounds: int = 3, f0: float = 20.0, b: float = 2.0, sclap_seq: bool = False) -> List[Level]:
    """Matching-based hierarchy (Q16/Q17) or SCLaP (sclap=True):
    the synchronous reading R6 (the GPU's rule), or with sclap_seq=True the
    paper's sequential random-order label propagation (R6s); contraction per
    P:225-232."""
    rp = np.ascontiguousarray(g.row_ptr, dtype=np.int64)
    col = np.ascontiguousarray(g.col, dtype=np.int32)
    om = None if omega is None else np.ascontiguousarray(omega, dtype=np.int64)
    cc = None if c is None else np.ascontiguousarray(c, dtype=np.int64)
    h = ctypes.c_void_p()
    L = lib()
    if sclap:
        _check(L.or_build_hierarchy_sclap_mode(g.n, _p(rp, ctypes.c_int64), _p(col, ctypes.c_int32),
                                               _p(om, ctypes.c_int64), _p(cc, ctypes.c_int64), seed, n_stop,
                                               max_levels, lp_rounds, f0, b, 1 if sclap_seq else 0,
                                               ctypes.byref(h)), "build_hierarchy_sclap")
    else:
        _check(L.or_build_hierarchy(g.n, _p(rp, ctypes.c_int64), _p(col, ctypes.c_int32),
                                    _p(om, ctypes.c_int64), _p(cc, ctypes.c_int64), seed, n_stop,
                                    max_levels, max_rounds, ctypes.byref(h)), "build_hierarchy")
    try:
        levels = []
        for l in range(L.or_hier_num_levels(h)):
            n = ctypes.c_int32(); nnz = ctypes.c_int64(); rounds = ctypes.c_int32()
            prp = _i64p(); pcol = _i32p(); pom = _i64p(); pc = _i64p(); ppar = _i32p()
            _check(L.or_hier_level(h, l, ctypes.byref(n), ctypes.byref(nnz), ctypes.byref(prp),
                                   ctypes.byref(pcol), ctypes.byref(pom), ctypes.byref(pc),
                                   ctypes.byref(ppar), ctypes.byref(rounds)), "hier_level")
            nn, mm = n.value, nnz.value
            par = None
            if ppar:
                par = np.ctypeslib.as_array(ppar, shape=(nn,)).copy() if nn else np.zeros(0, np.int32)
            levels.append(Level(
                n=nn,
                row_ptr=np.ctypeslib.as_array(prp, shape=(nn + 1,)).copy(),
                col=np.ctypeslib.as_array(pcol, shape=(mm,)).copy() if mm else np.zeros(0, np.int32),
                omega=np.ctypeslib.as_array(pom, shape=(mm,)).copy() if mm else np.zeros(0, np.int64),
                c=np.ctypeslib.as_array(pc, shape=(nn,)).copy(),
                parent=par, rounds=rounds.value))
        return levels
    finally:
        L.or_hier_free(h)


def ancestor(levels: List[Level], l: int, hp: int) -> np.ndarray:
    """H = parent_{l+hp-1} o ... o parent_l."""
    a = np.arange(levels[l].n, dtype=np.int32)
    for t in range(hp):
        a = levels[l + t].parent[a]
    return a


@dataclass
class CoarseS:
    row_ptr: np.ndarray
    col: np.ndarray
    d: np.ndarray
    w: np.ndarray


def coarse_sset(level: Level, dim: int) -> CoarseS:
    """Q7 / P:247-248: S = E^l, d = c_u^(1/dim) + c_v^(1/dim), w = d^-2."""
    rp = np.ascontiguousarray(level.row_ptr, dtype=np.int64)
    col = np.ascontiguousarray(level.col, dtype=np.int32)
    c = np.ascontiguousarray(level.c, dtype=np.int64)
    m = col.shape[0]
    d = np.empty(m, dtype=np.float64)
    w = np.empty(m, dtype=np.float64)
    _check(lib().or_coarse_sset(level.n, m, _p(rp, ctypes.c_int64), _p(col, ctypes.c_int32),
                                _p(c, ctypes.c_int64), dim, _p(d, ctypes.c_double), _p(w, ctypes.c_double)),
           "coarse_sset")
    return CoarseS(rp, col, d, w)


def init_box(n: int, dim: int, box: float, seed: int, level: int) -> np.ndarray:
    x = np.empty((n, dim), dtype=np.float64)
    _check(lib().or_init_box(n, dim, box, seed, level, _p(x, ctypes.c_double)), "init_box")
    return x


def prolong(parent: np.ndarray, xc: np.ndarray, seed: int, level: int) -> np.ndarray:
    parent = np.ascontiguousarray(parent, dtype=np.int32)
    xc = np.ascontiguousarray(xc, dtype=np.float64)
    n, dim = parent.shape[0], xc.shape[1]
    x = np.empty((n, dim), dtype=np.float64)
    _check(lib().or_prolong(n, dim, _p(parent, ctypes.c_int32), _p(xc, ctypes.c_double), seed, level,
                            _p(x, ctypes.c_double)), "prolong")
    return x


def prolong_disc(parent: np.ndarray, xc: np.ndarray, c_coarse: np.ndarray, seed: int, level: int) -> np.ndarray:
    """The paper's disc prolongation (reading R7): angle 2 pi U0,
    distance c(parent)^(1/dim) U1 (dim 3: direction from z = 2 U2 - 1)."""
    parent = np.ascontiguousarray(parent, dtype=np.int32)
    xc = np.ascontiguousarray(xc, dtype=np.float64)
    cc = np.ascontiguousarray(c_coarse, dtype=np.int64)
    n, dim = parent.shape[0], xc.shape[1]
    x = np.empty((n, dim), dtype=np.float64)
    _check(lib().or_prolong_disc(n, dim, _p(parent, ctypes.c_int32), _p(xc, ctypes.c_double),
                                 _p(cc, ctypes.c_int64), seed, level, _p(x, ctypes.c_double)), "prolong_disc")
    return x


def layout(g, S, dim: int, alpha: float, q: float, h: int, sweeps, seed: int, n_stop: int = 1000,
           x_init: Optional[np.ndarray] = None, nthreads: Optional[int] = None):
    """Multilevel driver (P:195-257 with fixed alpha).  Returns (x0, (stress, entropy, total), levels)."""
    rp = np.ascontiguousarray(g.row_ptr, dtype=np.int64)
    col = np.ascontiguousarray(g.col, dtype=np.int32)
    srp, scol, d, w = _csr(S)
    sw = np.ascontiguousarray(np.atleast_1d(sweeps), dtype=np.int32)
    xi = None if x_init is None else np.ascontiguousarray(x_init, dtype=np.float64)
    n = g.n
    out = np.empty((n, dim), dtype=np.float64)
    en = np.zeros(3, dtype=np.float64)
    nl = ctypes.c_int32()
    _check(lib().or_layout(n, dim, _p(rp, ctypes.c_int64), _p(col, ctypes.c_int32), _p(srp, ctypes.c_int64),
                           _p(scol, ctypes.c_int32), _p(d, ctypes.c_double), _p(w, ctypes.c_double), alpha, q, h,
                           _p(sw, ctypes.c_int32), sw.shape[0], seed, n_stop, _p(xi, ctypes.c_double),
                           _p(out, ctypes.c_double), _p(en, ctypes.c_double), ctypes.byref(nl),
                           nthreads or default_threads()), "layout")
    return out, (float(en[0]), float(en[1]), float(en[2])), nl.value


def layout_schedule(g, S, dim: int, q: float, h: int, sched: Schedule, seed: int, n_stop: int = 1000,
                    multilevel: bool = True, dynamic: bool = False, x_init: Optional[np.ndarray] = None,
                    nthreads: Optional[int] = None, sclap: bool = False, disc: bool = False,
                    sclap_seq: bool = False):
    """The paper's schedule or the dynamic update;
    sclap_seq: SCLaP by the paper's sequential label propagation (R6s).
    Returns (x0, (stress, entropy, total at alpha_min), levels, sweeps per level)."""
    rp = np.ascontiguousarray(g.row_ptr, dtype=np.int64)
    col = np.ascontiguousarray(g.col, dtype=np.int32)
    srp, scol, d, w = _csr(S)
    xi = None if x_init is None else np.ascontiguousarray(x_init, dtype=np.float64)
    n = g.n
    out = np.empty((n, dim), dtype=np.float64)
    en = np.zeros(3, dtype=np.float64)
    nl = ctypes.c_int32()
    sw = np.zeros(64, dtype=np.int32)
    flags = ((1 if multilevel else 0) | (2 if dynamic else 0) | (4 if sclap else 0) | (8 if disc else 0)
             | (16 if sclap_seq else 0))
    _check(lib().or_layout_schedule(n, dim, _p(rp, ctypes.c_int64), _p(col, ctypes.c_int32), _p(srp, ctypes.c_int64),
                                    _p(scol, ctypes.c_int32), _p(d, ctypes.c_double), _p(w, ctypes.c_double), q, h,
                                    ctypes.byref(sched), seed, n_stop, flags, _p(xi, ctypes.c_double),
                                    _p(out, ctypes.c_double), _p(en, ctypes.c_double), ctypes.byref(nl),
                                    _p(sw, ctypes.c_int32), nthreads or default_threads()), "layout_schedule")
    return out, (float(en[0]), float(en[1]), float(en[2])), nl.value, sw[:nl.value].copy()


def full_stress(g, x: np.ndarray, nthreads: Optional[int] = None):
    """F(x), the optimal scale s* and F(s* x) over unordered pairs.
    Returns (F, s_opt, F_opt, pairs)."""
    rp = np.ascontiguousarray(g.row_ptr, dtype=np.int64)
    col = np.ascontiguousarray(g.col, dtype=np.int32)
    x = np.ascontiguousarray(x, dtype=np.float64)
    n, dim = x.shape
    out = np.zeros(4, dtype=np.float64)
    _check(lib().or_full_stress(n, _p(rp, ctypes.c_int64), _p(col, ctypes.c_int32), dim, _p(x, ctypes.c_double),
                                _p(out, ctypes.c_double), nthreads or default_threads()), "full_stress")
    return float(out[0]), float(out[1]), float(out[2]), int(out[3])


def sclap_labels(g, U: int, rounds: int, seed: int, level: int, omega=None, c=None, seq: bool = False) -> np.ndarray:
    """One SCLaP clustering with size bound U (R6, or seq=True: the paper's
    sequential label propagation R6s); returns the labels."""
    rp = np.ascontiguousarray(g.row_ptr, dtype=np.int64)
    col = np.ascontiguousarray(g.col, dtype=np.int32)
    om = np.ascontiguousarray(np.ones(col.shape[0]) if omega is None else omega, dtype=np.int64)
    cc = np.ascontiguousarray(np.ones(g.n) if c is None else c, dtype=np.int64)
    lab = np.empty(g.n, dtype=np.int32)
    fn = lib().or_sclap_labels_seq if seq else lib().or_sclap_labels
    _check(fn(g.n, _p(rp, ctypes.c_int64), _p(col, ctypes.c_int32), _p(om, ctypes.c_int64),
              _p(cc, ctypes.c_int64), U, rounds, seed, level, _p(lab, ctypes.c_int32)), "sclap_labels")
    return lab
