"""Thin ctypes binding of libmm_b200.so (include/mm.h).

Argument marshalling only: every step of the hot path runs in the library's
sm_100a kernels.  Torch is used for device memory and streams (the current
stream of the tensors' device).  There is no CPU fallback: if the library or
a CUDA device is missing, calls raise.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MM_LIB_PATH") or os.path.join(_HERE, "libmm_b200.so")  # override: experiments only

MM_OK, MM_ERR_INVALID_ARGUMENT, MM_ERR_INVALID_INPUT, MM_ERR_NONFINITE = 0, -1, -2, -3
MM_ERR_OUT_OF_MEMORY, MM_ERR_CUDA, MM_ERR_UNSUPPORTED = -4, -5, -6
MM_MAX_LEVELS = 64

EXPORTS = ["mm_status_string", "mm_last_error", "mm_version", "mm_set_allocator", "mm_validate_sset",
           "mm_sweep_workspace", "mm_prolong", "mm_sweeps",
           "mm_sweep", "mm_energy", "mm_build_hierarchy", "mm_build_hierarchy_sclap", "mm_hierarchy_num_levels", "mm_hierarchy_level",
           "mm_hierarchy_free", "mm_hierarchy_copy_level", "mm_layout", "mm_layout_schedule", "mm_full_stress",
           "mm_launch_count", "mm_exact_kernel_variant",
           "mm_profile_enable",
           "mm_profile_reset", "mm_profile_read", "mm_profile_last"]


class MMError(RuntimeError):
    def __init__(self, status: int, where: str, detail: str):
        super().__init__(f"{where}: {status_name(status)}: {detail}")
        self.status = status


# ------------------------------------------------------------------ C structs
class mm_graph(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int32), ("nnz", ctypes.c_int64), ("row_ptr", ctypes.c_void_p),
                ("col", ctypes.c_void_p), ("omega", ctypes.c_void_p)]


class mm_sset(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int32), ("nnz", ctypes.c_int64), ("row_ptr", ctypes.c_void_p),
                ("col", ctypes.c_void_p), ("d", ctypes.c_void_p), ("w", ctypes.c_void_p)]


class mm_approx(ctypes.Structure):
    _fields_ = [("k", ctypes.c_int32), ("parent", ctypes.c_void_p), ("ancestor", ctypes.c_void_p)]


class mm_sweep_stats(ctypes.Structure):
    _fields_ = [("dx2", ctypes.c_double), ("x2", ctypes.c_double), ("stress", ctypes.c_double),
                ("flags", ctypes.c_int32), ("pad", ctypes.c_int32)]


class mm_level_view(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int32), ("nnz", ctypes.c_int64), ("row_ptr", ctypes.c_void_p),
                ("col", ctypes.c_void_p), ("omega", ctypes.c_void_p), ("c", ctypes.c_void_p),
                ("parent", ctypes.c_void_p), ("d", ctypes.c_void_p), ("w", ctypes.c_void_p),
                ("rounds", ctypes.c_int32)]


class mm_layout_report(ctypes.Structure):
    _fields_ = [("levels", ctypes.c_int32), ("n_level", ctypes.c_int32 * MM_MAX_LEVELS),
                ("k_level", ctypes.c_int32 * MM_MAX_LEVELS), ("stress", ctypes.c_double),
                ("entropy", ctypes.c_double), ("energy", ctypes.c_double), ("rel_change", ctypes.c_double),
                ("vertex_updates", ctypes.c_int64), ("pair_interactions", ctypes.c_int64),
                ("coincident_pairs", ctypes.c_int64), ("sweeps_level", ctypes.c_int32 * MM_MAX_LEVELS)]


class mm_schedule(ctypes.Structure):
    _fields_ = [("alpha0", ctypes.c_double), ("alpha_min", ctypes.c_double), ("factor", ctypes.c_double),
                ("eps", ctypes.c_double), ("a", ctypes.c_int32), ("max_final_iters", ctypes.c_int32)]


MM_LAYOUT_MULTILEVEL, MM_LAYOUT_DYNAMIC, MM_LAYOUT_SCLAP, MM_LAYOUT_DISC_PROLONG = 1, 2, 4, 8


def paper_schedule(**kw) -> mm_schedule:
    """The paper's defaults; max_final_iters is a safety cap."""
    v = dict(alpha0=1.0, alpha_min=0.008, factor=0.3, eps=1e-4, a=2, max_final_iters=200)
    v.update(kw)
    return mm_schedule(**v)


class mm_kernel_profile(ctypes.Structure):
    _fields_ = [("name", ctypes.c_char * 48), ("launches", ctypes.c_int64), ("total_ms", ctypes.c_double)]


_lib: Optional[ctypes.CDLL] = None


def load() -> ctypes.CDLL:
    """Load libmm_b200.so (fails loudly if it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
    L = ctypes.CDLL(LIB_PATH)
    vp, i32, i64, f32, f64, u64 = (ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_float,
                                  ctypes.c_double, ctypes.c_uint64)
    P = ctypes.POINTER
    L.mm_status_string.argtypes = [ctypes.c_int]; L.mm_status_string.restype = ctypes.c_char_p
    L.mm_last_error.argtypes = []; L.mm_last_error.restype = ctypes.c_char_p
    L.mm_version.argtypes = []; L.mm_version.restype = ctypes.c_char_p
    L.mm_set_allocator.argtypes = [vp, vp, vp]; L.mm_set_allocator.restype = ctypes.c_int
    L.mm_validate_sset.argtypes = [P(mm_sset), vp]; L.mm_validate_sset.restype = ctypes.c_int
    L.mm_sweeps.argtypes = [P(mm_sset), ctypes.c_int, f32, f32, P(mm_approx), vp, vp, i32, vp, vp]
    L.mm_sweeps.restype = ctypes.c_int
    L.mm_prolong.argtypes = [i32, ctypes.c_int, vp, vp, vp, u64, i32, vp, vp]
    L.mm_prolong.restype = ctypes.c_int
    L.mm_sweep_workspace.argtypes = [i32, ctypes.c_int, P(mm_approx), P(ctypes.c_size_t)]
    L.mm_sweep_workspace.restype = ctypes.c_int
    L.mm_sweep.argtypes = [P(mm_sset), ctypes.c_int, f32, f32, P(mm_approx), vp, vp, vp, vp, ctypes.c_size_t, vp]
    L.mm_sweep.restype = ctypes.c_int
    L.mm_energy.argtypes = [P(mm_sset), ctypes.c_int, f64, f64, vp, P(f64), vp]
    L.mm_energy.restype = ctypes.c_int
    L.mm_build_hierarchy.argtypes = [P(mm_graph), vp, ctypes.c_int, u64, i32, i32, i32, P(vp), vp]
    L.mm_build_hierarchy.restype = ctypes.c_int
    L.mm_build_hierarchy_sclap.argtypes = [P(mm_graph), vp, ctypes.c_int, u64, i32, i32, i32, f64, f64, P(vp), vp]
    L.mm_build_hierarchy_sclap.restype = ctypes.c_int
    L.mm_hierarchy_num_levels.argtypes = [vp]; L.mm_hierarchy_num_levels.restype = i32
    L.mm_hierarchy_level.argtypes = [vp, i32, P(mm_level_view)]; L.mm_hierarchy_level.restype = ctypes.c_int
    L.mm_hierarchy_free.argtypes = [vp]; L.mm_hierarchy_free.restype = None
    L.mm_hierarchy_copy_level.argtypes = [vp, i32, vp, vp, vp, vp, vp, vp, vp, vp]
    L.mm_hierarchy_copy_level.restype = ctypes.c_int
    L.mm_layout.argtypes = [P(mm_graph), P(mm_sset), ctypes.c_int, f32, f32, ctypes.c_int, P(i32), i32, u64, i32,
                            vp, vp, P(mm_layout_report), vp]
    L.mm_layout.restype = ctypes.c_int
    L.mm_layout_schedule.argtypes = [P(mm_graph), P(mm_sset), ctypes.c_int, f32, ctypes.c_int, P(mm_schedule), u64, i32,
                                     i32, vp, vp, P(mm_layout_report), vp]
    L.mm_layout_schedule.restype = ctypes.c_int
    L.mm_full_stress.argtypes = [P(mm_graph), ctypes.c_int, vp, P(f64), vp]
    L.mm_full_stress.restype = ctypes.c_int
    L.mm_launch_count.argtypes = []; L.mm_launch_count.restype = i64
    L.mm_exact_kernel_variant.argtypes = [i32, ctypes.c_int]; L.mm_exact_kernel_variant.restype = ctypes.c_int
    L.mm_profile_enable.argtypes = [ctypes.c_int]; L.mm_profile_enable.restype = ctypes.c_int
    L.mm_profile_reset.argtypes = []; L.mm_profile_reset.restype = ctypes.c_int
    L.mm_profile_read.argtypes = [P(mm_kernel_profile), i32, P(i32)]; L.mm_profile_read.restype = ctypes.c_int
    L.mm_profile_last.argtypes = [ctypes.c_char_p, i32, P(f64), P(i32)]; L.mm_profile_last.restype = ctypes.c_int
    _lib = L
    return L


def status_name(s: int) -> str:
    return load().mm_status_string(s).decode()


def _check(rc: int, where: str):
    if rc != MM_OK:
        raise MMError(rc, where, load().mm_last_error().decode())


def _torch():
    import torch
    return torch


def _stream_ptr(device=None) -> int:
    torch = _torch()
    return int(torch.cuda.current_stream(device).cuda_stream)


def _ptr(t) -> Optional[int]:
    return None if t is None else int(t.data_ptr())


# ------------------------------------------------------------------ device containers
@dataclass
class DeviceGraph:
    row_ptr: "object"
    col: "object"
    omega: "object" = None

    @property
    def n(self) -> int:
        return int(self.row_ptr.shape[0] - 1)

    def c_struct(self) -> mm_graph:
        return mm_graph(self.n, int(self.col.shape[0]), _ptr(self.row_ptr), _ptr(self.col), _ptr(self.omega))


@dataclass
class DeviceSSet:
    row_ptr: "object"
    col: "object"
    d: "object"
    w: "object"

    @property
    def n(self) -> int:
        return int(self.row_ptr.shape[0] - 1)

    @property
    def nnz(self) -> int:
        return int(self.col.shape[0])

    def c_struct(self) -> mm_sset:
        return mm_sset(self.n, self.nnz, _ptr(self.row_ptr), _ptr(self.col), _ptr(self.d), _ptr(self.w))


def graph_to_device(g, device="cuda", omega: Optional[np.ndarray] = None) -> DeviceGraph:
    torch = _torch()
    return DeviceGraph(torch.from_numpy(np.ascontiguousarray(g.row_ptr, dtype=np.int64)).to(device),
                       torch.from_numpy(np.ascontiguousarray(g.col, dtype=np.int32)).to(device),
                       None if omega is None else torch.from_numpy(np.ascontiguousarray(omega, np.int32)).to(device))


def sset_to_device(S, device="cuda") -> DeviceSSet:
    torch = _torch()
    return DeviceSSet(torch.from_numpy(np.ascontiguousarray(S.row_ptr, dtype=np.int64)).to(device),
                      torch.from_numpy(np.ascontiguousarray(S.col, dtype=np.int32)).to(device),
                      torch.from_numpy(np.ascontiguousarray(S.d, dtype=np.float32)).to(device),
                      torch.from_numpy(np.ascontiguousarray(S.w, dtype=np.float32)).to(device))


def coords_layout(x: np.ndarray) -> np.ndarray:
    """(n, dim) -> the library's layout: float32 (n, 2) for dim 2, (n, 4) for dim 3."""
    x = np.asarray(x, dtype=np.float32)
    n, dim = x.shape
    if dim == 2:
        return np.ascontiguousarray(x)
    out = np.zeros((n, 4), dtype=np.float32)
    out[:, :3] = x
    return out


def coords_to_device(x: np.ndarray, device="cuda"):
    torch = _torch()
    return torch.from_numpy(coords_layout(x)).to(device)


def coords_from_device(xt, dim: int) -> np.ndarray:
    return xt.detach().cpu().numpy()[:, :dim].astype(np.float64)


def _dim_of(xt) -> int:
    return 2 if xt.shape[1] == 2 else 3


# ------------------------------------------------------------------ API
def sweep_workspace(n: int, dim: int, k: int = 0) -> int:
    """Scratch bytes mm_sweep needs (k > 0: Eq.(3) with k representatives)."""
    b = ctypes.c_size_t(0)
    ap = mm_approx(int(k), None, None) if k > 0 else None
    _check(load().mm_sweep_workspace(int(n), int(dim), ctypes.byref(ap) if ap else None, ctypes.byref(b)),
           "mm_sweep_workspace")
    return int(b.value)


def sweep(S: DeviceSSet, x, alpha: float, q: float, parent=None, ancestor=None, k: int = 0,
          out=None, stats: bool = False, workspace=None):
    """One Jacobi sweep (Eq.(2), or Eq.(3) when parent/ancestor/k are given).
    x: CUDA float32 tensor (n,2) or (n,4).  workspace: optional CUDA uint8 tensor
    of at least sweep_workspace() bytes (else the library allocates).
    Returns x_out (and the stats dict)."""
    torch = _torch()
    L = load()
    dim = _dim_of(x)
    if out is None:
        out = torch.empty_like(x)
    st = None
    if stats:
        st = torch.zeros(4, dtype=torch.float64, device=x.device)  # 32 bytes = mm_sweep_stats
    ap = None
    if parent is not None:
        ap = mm_approx(int(k), _ptr(parent), _ptr(ancestor))
    s = S.c_struct()
    ws, wsb = (None, 0) if workspace is None else (_ptr(workspace), workspace.numel() * workspace.element_size())
    rc = L.mm_sweep(ctypes.byref(s), dim, float(alpha), float(q), ctypes.byref(ap) if ap else None,
                    _ptr(x), _ptr(out), _ptr(st), ws, wsb, _stream_ptr(x.device))
    _check(rc, "mm_sweep")
    if stats:
        h = st.cpu().numpy()
        flags = int(np.frombuffer(h[3:4].tobytes(), dtype=np.int32)[0])
        return out, {"dx2": float(h[0]), "x2": float(h[1]), "stress": float(h[2]), "flags": flags}
    return out


def sweeps(S: DeviceSSet, x, alpha: float, q: float, K: int, parent=None, ancestor=None, k: int = 0,
           out=None, stats: bool = False):
    """mm_sweeps: K Jacobi sweeps (Eq.(2), or Eq.(3) with parent/ancestor/k)
    from x; small levels run in the persistent kernel as in mm_layout."""
    torch = _torch()
    dim = _dim_of(x)
    if out is None:
        out = torch.empty_like(x)
    st = torch.zeros(4, dtype=torch.float64, device=x.device) if stats else None
    ap = mm_approx(int(k), _ptr(parent), _ptr(ancestor)) if parent is not None else None
    s = S.c_struct()
    rc = load().mm_sweeps(ctypes.byref(s), dim, float(alpha), float(q), ctypes.byref(ap) if ap else None,
                          _ptr(x), _ptr(out), int(K), _ptr(st), _stream_ptr(x.device))
    _check(rc, "mm_sweeps")
    if stats:
        h = st.cpu().numpy()
        flags = int(np.frombuffer(h[3:4].tobytes(), dtype=np.int32)[0])
        return out, {"dx2": float(h[0]), "x2": float(h[1]), "stress": float(h[2]), "flags": flags}
    return out


def energy(S: DeviceSSet, x, alpha: float, q: float):
    """Maxent-stress energy Eq.(1): (stress, entropy, total)."""
    L = load()
    out = (ctypes.c_double * 3)()
    s = S.c_struct()
    rc = L.mm_energy(ctypes.byref(s), _dim_of(x), float(alpha), float(q), _ptr(x), out, _stream_ptr(x.device))
    _check(rc, "mm_energy")
    return float(out[0]), float(out[1]), float(out[2])


class Hierarchy:
    """Owning handle of an mm_hierarchy (device storage, library-owned)."""

    def __init__(self, handle: int):
        self._h = ctypes.c_void_p(handle)

    def __del__(self):
        try:
            if self._h:
                load().mm_hierarchy_free(self._h)
                self._h = ctypes.c_void_p()
        except Exception:
            pass

    @property
    def num_levels(self) -> int:
        return int(load().mm_hierarchy_num_levels(self._h))

    def view(self, level: int) -> mm_level_view:
        v = mm_level_view()
        _check(load().mm_hierarchy_level(self._h, level, ctypes.byref(v)), "mm_hierarchy_level")
        return v

    def level_host(self, level: int) -> dict:
        """Copy one level to numpy arrays."""
        v = self.view(level)
        n, m = v.n, v.nnz
        rp = np.zeros(n + 1, np.int64)
        col = np.zeros(max(m, 1), np.int32)
        om = np.zeros(max(m, 1), np.int32)
        c = np.zeros(n, np.int32)
        par = np.zeros(n, np.int32) if v.parent else None
        d = np.zeros(max(m, 1), np.float32) if v.d else None
        w = np.zeros(max(m, 1), np.float32) if v.w else None
        ptr = lambda a: None if a is None else a.ctypes.data
        _check(load().mm_hierarchy_copy_level(self._h, level, ptr(rp), ptr(col), ptr(om), ptr(c), ptr(par),
                                              ptr(d), ptr(w), _stream_ptr()), "mm_hierarchy_copy_level")
        return {"n": n, "nnz": m, "row_ptr": rp, "col": col[:m], "omega": om[:m], "c": c, "parent": par,
                "d": None if d is None else d[:m], "w": None if w is None else w[:m], "rounds": v.rounds}


def build_hierarchy(g: DeviceGraph, dim: int, seed: int, n_stop: int = 1000, max_levels: int = 64,
                    max_rounds: int = 64, c=None, sclap: bool = False, lp_rounds: int = 3, f0: float = 20.0,
                    b: float = 2.0) -> Hierarchy:
    L = load()
    h = ctypes.c_void_p()
    gs = g.c_struct()
    if sclap:
        rc = L.mm_build_hierarchy_sclap(ctypes.byref(gs), _ptr(c), dim, seed, n_stop, max_levels, lp_rounds, f0, b,
                                        ctypes.byref(h), _stream_ptr(g.row_ptr.device))
        _check(rc, "mm_build_hierarchy_sclap")
    else:
        rc = L.mm_build_hierarchy(ctypes.byref(gs), _ptr(c), dim, seed, n_stop, max_levels, max_rounds,
                                  ctypes.byref(h), _stream_ptr(g.row_ptr.device))
        _check(rc, "mm_build_hierarchy")
    return Hierarchy(h.value)


def layout(g: Optional[DeviceGraph], S: DeviceSSet, dim: int, alpha: float, q: float, h: int,
           sweeps: Sequence[int], seed: int, n_stop: int = 1000, x_init=None, out=None):
    """Multilevel (h > 0) or single-level exact (h = 0, x_init required) layout.
    Returns (x_out tensor, report dict)."""
    torch = _torch()
    L = load()
    n = S.n
    device = S.row_ptr.device
    if out is None:
        out = torch.empty((n, 2 if dim == 2 else 4), dtype=torch.float32, device=device)
    sw = (ctypes.c_int32 * len(sweeps))(*[int(k) for k in sweeps])
    rep = mm_layout_report()
    gs = g.c_struct() if g is not None else None
    s = S.c_struct()
    rc = L.mm_layout(ctypes.byref(gs) if gs is not None else None, ctypes.byref(s), dim, float(alpha), float(q),
                     int(h), sw, len(sweeps), int(seed), int(n_stop), _ptr(x_init), _ptr(out), ctypes.byref(rep),
                     _stream_ptr(device))
    _check(rc, "mm_layout")
    return out, _report(rep)


def _report(rep: mm_layout_report) -> dict:
    return {"levels": rep.levels, "n_level": list(rep.n_level[:rep.levels]),
            "k_level": list(rep.k_level[:rep.levels]), "sweeps_level": list(rep.sweeps_level[:rep.levels]),
            "stress": rep.stress, "entropy": rep.entropy, "energy": rep.energy, "rel_change": rep.rel_change,
            "vertex_updates": rep.vertex_updates, "pair_interactions": rep.pair_interactions,
            "coincident_pairs": rep.coincident_pairs}


def layout_schedule(g: Optional[DeviceGraph], S: DeviceSSet, dim: int, q: float, h: int, sched: mm_schedule,
                    seed: int, n_stop: int = 1000, multilevel: bool = True, dynamic: bool = False, x_init=None,
                    out=None, sclap: bool = False, disc: bool = False):
    """The paper's alpha schedule or the dynamic update.
    Returns (x_out tensor, report dict incl. sweeps_level)."""
    torch = _torch()
    L = load()
    n = S.n
    device = S.row_ptr.device
    if out is None:
        out = torch.empty((n, 2 if dim == 2 else 4), dtype=torch.float32, device=device)
    rep = mm_layout_report()
    gs = g.c_struct() if g is not None else None
    s = S.c_struct()
    flags = ((MM_LAYOUT_MULTILEVEL if multilevel else 0) | (MM_LAYOUT_DYNAMIC if dynamic else 0) |
             (MM_LAYOUT_SCLAP if sclap else 0) | (MM_LAYOUT_DISC_PROLONG if disc else 0))
    rc = L.mm_layout_schedule(ctypes.byref(gs) if gs is not None else None, ctypes.byref(s), dim, float(q), int(h),
                              ctypes.byref(sched), int(seed), int(n_stop), flags, _ptr(x_init), _ptr(out),
                              ctypes.byref(rep), _stream_ptr(device))
    _check(rc, "mm_layout_schedule")
    return out, _report(rep)


def launch_count() -> int:
    return int(load().mm_launch_count())


def exact_kernel_variant(n: int, dim: int) -> int:
    """0: one-sided kernel (b); 1: symmetric kernel (b)."""
    return int(load().mm_exact_kernel_variant(int(n), int(dim)))


def profile_enable(on: bool = True):
    load().mm_profile_enable(1 if on else 0)


def profile_reset():
    load().mm_profile_reset()


def profile_read() -> dict:
    L = load()
    cnt = ctypes.c_int32()
    L.mm_profile_read(None, 0, ctypes.byref(cnt))
    arr = (mm_kernel_profile * max(cnt.value, 1))()
    L.mm_profile_read(arr, cnt.value, ctypes.byref(cnt))
    return {arr[i].name.decode(): {"launches": int(arr[i].launches), "total_ms": float(arr[i].total_ms)}
            for i in range(cnt.value)}


def profile_last(name: str, count: int) -> list:
    """Device ms of the last `count` timed launches of kernel `name` (launch order)."""
    ms = (ctypes.c_double * max(count, 1))()
    got = ctypes.c_int32()
    _check(load().mm_profile_last(name.encode(), int(count), ms, ctypes.byref(got)), "mm_profile_last")
    return [float(ms[i]) for i in range(got.value)]


def full_stress(g: DeviceGraph, x):
    """Full stress F(x), optimal scale s*, F(s* x), pair count."""
    L = load()
    out = (ctypes.c_double * 4)()
    gs = g.c_struct()
    _check(L.mm_full_stress(ctypes.byref(gs), _dim_of(x), _ptr(x), out, _stream_ptr(x.device)), "mm_full_stress")
    return float(out[0]), float(out[1]), float(out[2]), int(out[3])


def prolong(parent, xc, seed: int, level: int, c_coarse=None, out=None):
    """mm_prolong: x[u] = xc[parent[u]] + jitter (Q15) or the paper's disc
     when the coarse node weights c_coarse are given.  parent: CUDA
    int32 (n_fine,); xc: CUDA float32 coarse coordinates; level: the fine level."""
    torch = _torch()
    dim = _dim_of(xc)
    n = int(parent.shape[0])
    if out is None:
        out = torch.empty((n, xc.shape[1]), dtype=torch.float32, device=xc.device)
    rc = load().mm_prolong(n, dim, _ptr(parent), _ptr(xc), _ptr(c_coarse), int(seed) & 0xFFFFFFFFFFFFFFFF,
                           int(level), _ptr(out), _stream_ptr(xc.device))
    _check(rc, "mm_prolong")
    return out


def validate_sset(S: DeviceSSet):
    """Device-side validation of an S set (raises MMError(MM_ERR_INVALID_INPUT))."""
    s = S.c_struct()
    _check(load().mm_validate_sset(ctypes.byref(s), _stream_ptr(S.row_ptr.device)), "mm_validate_sset")
