"""paper_1705_02408_b200 -- B200-native MPAP hot path (arXiv 1705.02408).

Thin ctypes binding over ``libmpap.so`` (C ABI: ``include/mpap.h``).  The
functions below carry the ABI names and only marshal arguments: every step of
the roadmap build and of the search runs in the library's sm_100a kernels.
There is no CPU fallback -- importing this package raises if the in-tree
library is missing (build it with ``python build_ext.py``).

PyTorch is used only for device memory and streams: device-resident inputs
are passed as CUDA tensors (``mem = MPAP_MEM_DEVICE``), and the current torch
stream is handed to the library.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Any, Dict, Optional, Sequence

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MPAP_LIB") or os.path.join(_PKG, "libmpap.so")   # MPAP_LIB: tuning variants

if not os.path.exists(LIB_PATH):
    raise ImportError(f"libmpap.so not found at {LIB_PATH}: build it with "
                      "`python build_ext.py` (no CPU fallback exists)")

_lib = C.CDLL(LIB_PATH)

MPAP_OK = 0
MPAP_ERR_INVALID_ARGUMENT = 1
MPAP_ERR_NO_GOAL_NODE = 2
MPAP_ERR_NO_FEASIBLE_PLAN = 3
MPAP_ERR_BUFFER_TOO_SMALL = 4
MPAP_ERR_OUT_OF_MEMORY = 5
MPAP_ERR_CUDA = 6
STATUS_NAMES = {0: "OK", 1: "INVALID_ARGUMENT", 2: "NO_GOAL_NODE", 3: "NO_FEASIBLE_PLAN", 4: "BUFFER_TOO_SMALL",
                5: "OUT_OF_MEMORY", 6: "CUDA"}
MPAP_MEM_HOST = 0
MPAP_MEM_DEVICE = 1
MPAP_SEARCH_FORALL_T = 1

EXPORTED_SYMBOLS = [
    "mpap_build_roadmap_batch", "mpap_build_roadmap", "mpap_search", "mpap_search_batch", "mpap_roadmap_import",
    "mpap_roadmap_info", "mpap_roadmap_envs", "mpap_roadmap_export", "mpap_roadmap_free", "mpap_status_str",
    "mpap_last_error", "mpap_launch_count", "mpap_prof_enable", "mpap_prof_reset", "mpap_prof_read",
    "mpap_roadmap_work", "mpap_search_ex", "mpap_search_batch_ex", "mpap_roadmap_export_peaks",
    "mpap_roadmap_set_peaks", "mpap_roadmap_update", "mpap_mc_verify", "mpap_mc_verify_batch",
    "mpap_roadmap_rows_evaluated", "mpap_build_roadmap_rows", "mpap_prof_fp64_peak",
    "mpap_search_batch_trace", "mpap_search_launches", "mpap_roadmap_block_device",
    "mpap_roadmap_assemble_device",
]


class MpapError(RuntimeError):
    def __init__(self, status: int, where: str):
        self.status = status
        msg = _lib.mpap_last_error().decode(errors="replace")
        super().__init__(f"{where}: {STATUS_NAMES.get(status, status)}: {msg}")


class mpap_params(C.Structure):
    _fields_ = [
        ("pos_dim", C.c_int32), ("dynamics", C.c_int32), ("has_heading", C.c_int32), ("heuristic", C.c_int32),
        ("ws_lo", C.c_double * 3), ("ws_hi", C.c_double * 3),
        ("control_weight", C.c_double), ("nominal_speed", C.c_double), ("dt", C.c_double),
        ("collision_dt", C.c_double), ("n_f", C.c_double), ("fov_cos_half", C.c_double),
        ("max_range", C.c_double), ("mlp", C.POINTER(C.c_double)), ("mlp_gain", C.c_double),
        ("v_ref", C.c_double), ("w_ref", C.c_double), ("edge_peaks", C.c_int32), ("lazy_edges", C.c_int32),
    ]


class mpap_goal(C.Structure):
    _fields_ = [("lo", C.c_double * 3), ("hi", C.c_double * 3)]


class mpap_result(C.Structure):
    _fields_ = [
        ("status", C.c_int32), ("path_len", C.c_int32), ("waves", C.c_int32), ("retries", C.c_int32),
        ("cost", C.c_float), ("h", C.c_float), ("h_peak", C.c_float), ("pad", C.c_float),
        ("relaxations", C.c_int64), ("labels_inserted", C.c_int64),
    ]


WAVE_FIELDS = ["i", "group", "relax", "beta_pass", "inserted", "killed", "touched", "stair_sum"]


class mpap_wave(C.Structure):
    _fields_ = [(f, C.c_int64) for f in WAVE_FIELDS]


RESULT_DTYPE = np.dtype([("status", np.int32), ("path_len", np.int32), ("waves", np.int32), ("retries", np.int32),
                         ("cost", np.float32), ("h", np.float32), ("h_peak", np.float32), ("pad", np.float32),
                         ("relaxations", np.int64), ("labels_inserted", np.int64)])
assert RESULT_DTYPE.itemsize == C.sizeof(mpap_result) == 48

class mpap_mc_params(C.Structure):
    _fields_ = [("trials", C.c_int32), ("pad", C.c_int32), ("seed", C.c_uint64),
                ("sigma_imu", C.c_double), ("sigma_vis", C.c_double), ("u_max", C.c_double),
                ("k_p", C.c_double), ("k_d", C.c_double), ("p0_pos", C.c_double), ("p0_vel", C.c_double),
                ("delta", C.c_double)]


MC_RESULT_DTYPE = np.dtype([("status", np.int32), ("trials", np.int32), ("exceed", np.int64), ("steps", np.int64),
                            ("fixes", np.int64), ("p_hat", np.float64)])

_vp = C.c_void_p
_i32p = C.POINTER(C.c_int32)
_lib.mpap_build_roadmap_batch.argtypes = [C.c_int32, _vp, _i32p, C.c_int32, _vp, _i32p, _vp, _i32p, C.c_double,
                                          C.POINTER(mpap_params), C.c_int32, _vp, C.POINTER(_vp)]
_lib.mpap_build_roadmap.argtypes = [_vp, C.c_int32, C.c_int32, _vp, C.c_int32, _vp, C.c_int32, C.c_double,
                                    C.POINTER(mpap_params), C.c_int32, _vp, C.POINTER(_vp)]
_lib.mpap_search.argtypes = [_vp, C.c_int32, C.c_int32, C.POINTER(mpap_goal), C.c_double, C.c_double, _i32p,
                             C.c_int32, C.POINTER(mpap_result), C.POINTER(mpap_wave), C.c_int32, _vp]
_lib.mpap_search_batch.argtypes = [_vp, C.c_int32, _i32p, _i32p, C.POINTER(mpap_goal), C.POINTER(C.c_double),
                                   C.c_double, _vp, C.c_int32, _vp, C.c_int32, _vp]
_lib.mpap_search_ex.argtypes = [_vp, C.c_int32, C.c_int32, C.POINTER(mpap_goal), C.c_double, C.c_double, C.c_uint32,
                                _i32p, C.c_int32, C.POINTER(mpap_result), C.POINTER(mpap_wave), C.c_int32, _vp]
_lib.mpap_search_batch_ex.argtypes = [_vp, C.c_int32, _i32p, _i32p, C.POINTER(mpap_goal), C.POINTER(C.c_double),
                                      C.c_double, C.c_uint32, _vp, C.c_int32, _vp, C.c_int32, _vp]
if hasattr(_lib, "mpap_search_batch_trace"):   # (older tuning builds loaded via MPAP_LIB may lack it)
    _lib.mpap_search_batch_trace.argtypes = [_vp, C.c_int32, _i32p, _i32p, C.POINTER(mpap_goal),
                                             C.POINTER(C.c_double), C.c_double, C.c_uint32, _vp, C.c_int32, _vp,
                                             C.c_int32, _vp, C.c_int32, _vp]
_lib.mpap_mc_verify_batch.argtypes = [_vp, C.c_int32, _vp, _vp, C.c_int32, _vp, C.POINTER(mpap_mc_params),
                                      C.c_uint64, _vp, _vp, _vp, _vp]
_lib.mpap_mc_verify.argtypes = [_vp, C.c_int32, _vp, C.c_int32, C.POINTER(mpap_mc_params), C.c_uint64, _vp, _vp,
                                _vp, _vp]
_lib.mpap_build_roadmap_rows.argtypes = [_vp, C.c_int32, C.c_int32, _vp, C.c_int32, _vp, C.c_int32, C.c_double,
                                         C.POINTER(mpap_params), C.c_int32, C.c_int32, C.c_int32, _vp,
                                         C.POINTER(_vp)]
_lib.mpap_roadmap_rows_evaluated.argtypes = [_vp, C.c_int32, C.POINTER(C.c_int64)]
_lib.mpap_roadmap_export_peaks.argtypes = [_vp, C.c_int32, _vp, _vp]
_lib.mpap_roadmap_set_peaks.argtypes = [_vp, _vp, _vp]
_lib.mpap_roadmap_update.argtypes = [_vp, C.c_int32, _vp, C.c_int32, _vp, C.c_int32, C.c_int32, _vp,
                                     C.POINTER(C.c_int64)]
_lib.mpap_roadmap_import.argtypes = [C.c_int32, C.c_int32, _vp, _i32p, _vp, _vp, _vp, _vp, C.c_double, _vp,
                                     C.POINTER(_vp)]
_lib.mpap_roadmap_info.argtypes = [_vp, C.c_int32, _i32p, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
_lib.mpap_roadmap_work.argtypes = [_vp, C.POINTER(C.c_uint64), C.c_int32]
_lib.mpap_roadmap_work.restype = C.c_int
_lib.mpap_roadmap_envs.argtypes = [_vp]
_lib.mpap_roadmap_envs.restype = C.c_int32
_lib.mpap_roadmap_export.argtypes = [_vp, C.c_int32, _i32p, _vp, _vp, _vp, _vp]
_lib.mpap_roadmap_free.argtypes = [_vp]
_lib.mpap_roadmap_free.restype = None
_lib.mpap_status_str.argtypes = [C.c_int]
_lib.mpap_status_str.restype = C.c_char_p
_lib.mpap_last_error.restype = C.c_char_p
_lib.mpap_launch_count.restype = C.c_int64
_lib.mpap_prof_enable.argtypes = [C.c_int32]
_lib.mpap_prof_enable.restype = None
_lib.mpap_prof_reset.restype = None
_lib.mpap_prof_read.argtypes = [C.c_char_p, C.POINTER(C.c_double), C.POINTER(C.c_int64)]
_lib.mpap_prof_read.restype = C.c_int32
if hasattr(_lib, "mpap_roadmap_block_device"):
    _lib.mpap_roadmap_block_device.argtypes = [_vp, _vp, _vp, C.c_int64, C.POINTER(C.c_int64), _vp]
    _lib.mpap_roadmap_assemble_device.argtypes = [C.c_int32, C.c_int32, _vp, C.c_int32, _i32p, _vp, C.c_int32, _vp,
                                                  C.c_int64, C.c_double, _vp, C.POINTER(_vp)]
if hasattr(_lib, "mpap_prof_fp64_peak"):
    _lib.mpap_prof_fp64_peak.argtypes = [C.c_int32, C.POINTER(C.c_double), C.POINTER(C.c_double)]
    _lib.mpap_prof_fp64_peak.restype = C.c_int
if hasattr(_lib, "mpap_search_launches"):
    _lib.mpap_search_launches.argtypes = [C.c_int32]
    _lib.mpap_search_launches.restype = C.c_int64
for _f in ("mpap_build_roadmap_batch", "mpap_build_roadmap", "mpap_search", "mpap_search_batch",
           "mpap_search_ex", "mpap_search_batch_ex", "mpap_roadmap_export_peaks", "mpap_roadmap_set_peaks",
           "mpap_roadmap_update", "mpap_roadmap_import", "mpap_roadmap_info", "mpap_roadmap_export"):
    getattr(_lib, _f).restype = C.c_int


def lib():
    return _lib


def _stream(stream) -> Optional[int]:
    """cudaStream_t for the library: an explicit handle, a torch stream, or the
    current torch stream."""
    if stream is not None:
        return int(getattr(stream, "cuda_stream", stream))
    try:
        import torch
        if torch.cuda.is_available():
            return int(torch.cuda.current_stream().cuda_stream)
    except Exception:  # pragma: no cover
        pass
    return None


def _is_cuda_tensor(x) -> bool:
    return hasattr(x, "is_cuda") and bool(getattr(x, "is_cuda"))


def _ptr(x, dtype) -> Any:
    """(pointer, keepalive) for a numpy array or a contiguous torch tensor."""
    if _is_cuda_tensor(x):
        assert x.is_contiguous()
        return C.c_void_p(int(x.data_ptr())), x
    if hasattr(x, "data_ptr") and hasattr(x, "is_contiguous"):   # host torch tensor (e.g. pinned)
        assert x.is_contiguous() and x.element_size() == np.dtype(dtype).itemsize
        return C.c_void_p(int(x.data_ptr())), x
    a = np.ascontiguousarray(x, dtype=dtype)
    return C.c_void_p(a.ctypes.data if a.size else 0), a


class Roadmap:
    """Owning handle of a device-resident roadmap (mpap_roadmap*)."""

    def __init__(self, handle: int):
        self.handle = C.c_void_p(handle)

    def free(self):
        if self.handle:
            _lib.mpap_roadmap_free(self.handle)
            self.handle = C.c_void_p(0)

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass

    @property
    def envs(self) -> int:
        return int(_lib.mpap_roadmap_envs(self.handle))


def make_params(pos_dim: int, dynamics: int, has_heading: int, heuristic: int, ws_lo, ws_hi,
                mlp: Optional[np.ndarray], edge_peaks: bool = False, lazy_edges: bool = False,
                **p) -> mpap_params:
    """Pack an mpap_params struct (the MLP array must outlive the call that uses it).
    ``edge_peaks`` also computes the per-edge peaks MPAP_SEARCH_FORALL_T needs;
    ``lazy_edges`` defers collision + heuristic of each row to its first
    expansion by the single-query search (NEXT-1 part i)."""
    prm = mpap_params()
    prm.edge_peaks = 1 if edge_peaks else 0
    prm.lazy_edges = 1 if lazy_edges else 0
    prm.pos_dim, prm.dynamics, prm.has_heading, prm.heuristic = pos_dim, dynamics, has_heading, heuristic
    for k in range(3):
        prm.ws_lo[k] = float(ws_lo[k]) if k < len(ws_lo) else 0.0
        prm.ws_hi[k] = float(ws_hi[k]) if k < len(ws_hi) else 0.0
    for name in ("control_weight", "nominal_speed", "dt", "collision_dt", "n_f", "fov_cos_half", "max_range",
                 "mlp_gain", "v_ref", "w_ref"):
        setattr(prm, name, float(p[name]))
    if mlp is not None:
        prm.mlp = np.ascontiguousarray(mlp, dtype=np.float64).ctypes.data_as(C.POINTER(C.c_double))
    return prm


def params_from_problem(prob, edge_peaks: bool = False, lazy_edges: bool = False) -> tuple:
    """(mpap_params, keepalive) from a synth.Problem (marshalling only)."""
    mlp = np.ascontiguousarray(prob.mlp, dtype=np.float64)
    prm = make_params(prob.pos_dim, prob.dynamics, prob.has_heading, prob.heuristic, prob.ws_lo, prob.ws_hi,
                      mlp, edge_peaks=edge_peaks, lazy_edges=lazy_edges, **prob.params)
    return prm, mlp


def mpap_build_roadmap_batch(samples, n: Sequence[int], row_stride: int, obstacles, n_obstacles: Sequence[int],
                             features, n_features: Sequence[int], r: float, params: mpap_params,
                             stream=None) -> Roadmap:
    """Alg. 2 + heuristic precompute for a batch of environments.  ``samples``,
    ``obstacles``, ``features`` are numpy arrays (host) or CUDA tensors
    (device, float64, contiguous); the counts are host sequences."""
    dev = _is_cuda_tensor(samples)
    mem = MPAP_MEM_DEVICE if dev else MPAP_MEM_HOST
    sp, k1 = _ptr(samples, np.float64)
    op, k2 = _ptr(obstacles, np.float64)
    fp, k3 = _ptr(features, np.float64)
    na = np.ascontiguousarray(n, dtype=np.int32)
    oa = np.ascontiguousarray(n_obstacles, dtype=np.int32)
    fa = np.ascontiguousarray(n_features, dtype=np.int32)
    out = C.c_void_p()
    st = _stream(stream)
    s = _lib.mpap_build_roadmap_batch(len(na), sp, na.ctypes.data_as(_i32p), int(row_stride), op,
                                      oa.ctypes.data_as(_i32p), fp, fa.ctypes.data_as(_i32p), float(r),
                                      C.byref(params), mem, C.c_void_p(st) if st else None, C.byref(out))
    del k1, k2, k3
    if s != MPAP_OK:
        raise MpapError(s, "mpap_build_roadmap_batch")
    return Roadmap(out.value)


def mpap_build_roadmap(samples, obstacles, features, r: float, params: mpap_params, stream=None) -> Roadmap:
    """North-star form ``mpap_build_roadmap(samples, obstacles, features, r)``
    for one environment (arrays shaped [n, stride], [O, 2d], [F, d])."""
    n = int(samples.shape[0])
    stride = int(samples.shape[1])
    d = params.pos_dim
    no = int(obstacles.shape[0]) if obstacles is not None and np.size(obstacles) else 0
    nf = int(features.shape[0]) if features is not None and np.size(features) else 0
    dev = _is_cuda_tensor(samples)
    mem = MPAP_MEM_DEVICE if dev else MPAP_MEM_HOST
    sp, k1 = _ptr(samples, np.float64)
    op, k2 = _ptr(obstacles if no else np.zeros(2 * d), np.float64)
    fp, k3 = _ptr(features if nf else np.zeros(d), np.float64)
    out = C.c_void_p()
    st = _stream(stream)
    s = _lib.mpap_build_roadmap(sp, n, stride, op, no, fp, nf, float(r), C.byref(params), mem,
                                C.c_void_p(st) if st else None, C.byref(out))
    del k1, k2, k3
    if s != MPAP_OK:
        raise MpapError(s, "mpap_build_roadmap")
    return Roadmap(out.value)


def mpap_build_roadmap_rows(samples, obstacles, features, r: float, params: mpap_params, row_begin: int,
                            row_end: int, stream=None) -> Roadmap:
    """Row-sharded build: only rows [row_begin, row_end) of
    the single environment get edges; every sample is a candidate neighbour."""
    n = int(samples.shape[0])
    stride = int(samples.shape[1])
    d = params.pos_dim
    no = int(obstacles.shape[0]) if obstacles is not None and np.size(obstacles) else 0
    nf = int(features.shape[0]) if features is not None and np.size(features) else 0
    mem = MPAP_MEM_DEVICE if _is_cuda_tensor(samples) else MPAP_MEM_HOST
    sp, k1 = _ptr(samples, np.float64)
    op, k2 = _ptr(obstacles if no else np.zeros(2 * d), np.float64)
    fp, k3 = _ptr(features if nf else np.zeros(d), np.float64)
    out = C.c_void_p()
    st = _stream(stream)
    s = _lib.mpap_build_roadmap_rows(sp, n, stride, op, no, fp, nf, float(r), C.byref(params), int(row_begin),
                                     int(row_end), mem, C.c_void_p(st) if st else None, C.byref(out))
    del k1, k2, k3
    if s != MPAP_OK:
        raise MpapError(s, "mpap_build_roadmap_rows")
    return Roadmap(out.value)


def mpap_roadmap_import(positions, row_ptr, dst_coll, w, s, c, r: float, stream=None) -> Roadmap:
    pos = np.ascontiguousarray(positions, dtype=np.float64)
    n, d = pos.shape
    rp = np.ascontiguousarray(row_ptr, dtype=np.int32)
    dc = np.ascontiguousarray(dst_coll, dtype=np.uint32)
    wa = np.ascontiguousarray(w, dtype=np.float32)
    sa = np.ascontiguousarray(s, dtype=np.float32)
    ca = np.ascontiguousarray(c, dtype=np.float32)
    if dc.size == 0:
        dc, wa, sa, ca = np.zeros(1, np.uint32), np.zeros(1, np.float32), np.zeros(1, np.float32), \
            np.zeros(1, np.float32)
    out = C.c_void_p()
    st = _stream(stream)
    st_ = _lib.mpap_roadmap_import(n, d, pos.ctypes.data, rp.ctypes.data_as(_i32p), dc.ctypes.data, wa.ctypes.data,
                                   sa.ctypes.data, ca.ctypes.data, float(r), C.c_void_p(st) if st else None,
                                   C.byref(out))
    if st_ != MPAP_OK:
        raise MpapError(st_, "mpap_roadmap_import")
    return Roadmap(out.value)


def _goal(lo, hi) -> mpap_goal:
    g = mpap_goal()
    for k in range(3):
        g.lo[k] = float(lo[k]) if k < len(lo) else 0.0
        g.hi[k] = float(hi[k]) if k < len(hi) else 0.0
    return g


def mpap_search(rm: Roadmap, env: int, start: int, goal_lo, goal_hi, perception_bound: float, lam: float,
                path_capacity: int = 65536, trace_waves: int = 0, stream=None, forall_t: bool = False
                ) -> Dict[str, Any]:
    """Alg. 3 for one query; returns the plan, its cost and perception value
    (plus counters, and per-wave counters when ``trace_waves`` > 0).  A
    NO_FEASIBLE_PLAN outcome is returned, not raised.  ``forall_t`` selects
    MPAP_SEARCH_FORALL_T (Eq. 2 for every step along the edges)."""
    g = _goal(goal_lo, goal_hi)
    path = np.zeros(max(path_capacity, 1), dtype=np.int32)
    res = mpap_result()
    waves = (mpap_wave * trace_waves)() if trace_waves > 0 else None
    st = _stream(stream)
    s = _lib.mpap_search_ex(rm.handle, int(env), int(start), C.byref(g), float(perception_bound), float(lam),
                            MPAP_SEARCH_FORALL_T if forall_t else 0, path.ctypes.data_as(_i32p), int(path_capacity),
                            C.byref(res), waves, int(trace_waves), C.c_void_p(st) if st else None)
    if s not in (MPAP_OK, MPAP_ERR_NO_FEASIBLE_PLAN):
        raise MpapError(s, "mpap_search")
    out = {
        "status": int(res.status), "status_str": STATUS_NAMES.get(int(res.status), "?"),
        "path": path[: res.path_len].copy() if s == MPAP_OK else np.zeros(0, np.int32),
        "cost": np.float32(res.cost), "h": np.float32(res.h), "h_peak": np.float32(res.h_peak),
        "waves": int(res.waves), "relaxations": int(res.relaxations), "labels_inserted": int(res.labels_inserted),
        "retries": int(res.retries),
    }
    if waves is not None:
        nw = min(int(res.waves), trace_waves)
        out["wave_counters"] = np.array([[getattr(waves[k], f) for f in WAVE_FIELDS] for k in range(nw)],
                                        dtype=np.int64).reshape(-1, 8)
    return out


def mpap_search_batch(rm: Roadmap, envs, starts, goals_lo, goals_hi, perception_bounds, lam: float,
                      path_capacity: int, paths=None, results=None, stream=None, forall_t: bool = False,
                      trace_waves: int = 0):
    """Batch of independent queries (one CTA per query, dynamic scheduling).
    With ``paths``/``results`` CUDA tensors (int32 [Q, cap], uint8 [Q*48]) the
    call is asynchronous and writes on the device; otherwise host numpy outputs
    are returned.  ``trace_waves`` > 0 calls mpap_search_batch_trace and also
    returns the per-wave counters: (paths, results, [int64 [waves_q, 8] per
    query])."""
    Q = len(envs)
    ea = np.ascontiguousarray(envs, dtype=np.int32)
    sa = np.ascontiguousarray(starts, dtype=np.int32)
    ba = np.ascontiguousarray(perception_bounds, dtype=np.float64)
    gs = (mpap_goal * max(Q, 1))()
    for k in range(Q):
        gs[k] = _goal(goals_lo[k], goals_hi[k])
    st = _stream(stream)
    if paths is not None and _is_cuda_tensor(paths):
        mem = MPAP_MEM_DEVICE
        pp, rp = C.c_void_p(int(paths.data_ptr())), C.c_void_p(int(results.data_ptr()))
        host_paths = host_res = None
    else:
        mem = MPAP_MEM_HOST
        host_paths = np.zeros((Q, path_capacity), dtype=np.int32)
        host_res = np.zeros(Q, dtype=RESULT_DTYPE)
        pp, rp = C.c_void_p(host_paths.ctypes.data), C.c_void_p(host_res.ctypes.data)
    if trace_waves > 0:
        wv = np.zeros((max(Q, 1), trace_waves, 8), dtype=np.int64)
        s = _lib.mpap_search_batch_trace(rm.handle, Q, ea.ctypes.data_as(_i32p), sa.ctypes.data_as(_i32p), gs,
                                         ba.ctypes.data_as(C.POINTER(C.c_double)), float(lam),
                                         MPAP_SEARCH_FORALL_T if forall_t else 0, pp, int(path_capacity), rp, mem,
                                         C.c_void_p(wv.ctypes.data), int(trace_waves),
                                         C.c_void_p(st) if st else None)
        if s != MPAP_OK:
            raise MpapError(s, "mpap_search_batch_trace")
        res_h = host_res if host_res is not None else results.cpu().numpy().view(RESULT_DTYPE)
        counters = [wv[q, : min(int(res_h["waves"][q]), trace_waves)].copy() for q in range(Q)]
        return host_paths, host_res, counters
    s = _lib.mpap_search_batch_ex(rm.handle, Q, ea.ctypes.data_as(_i32p), sa.ctypes.data_as(_i32p), gs,
                                  ba.ctypes.data_as(C.POINTER(C.c_double)), float(lam),
                                  MPAP_SEARCH_FORALL_T if forall_t else 0, pp, int(path_capacity), rp, mem,
                                  C.c_void_p(st) if st else None)
    if s != MPAP_OK:
        raise MpapError(s, "mpap_search_batch")
    return host_paths, host_res


def mpap_roadmap_info(rm: Roadmap, env: int = 0) -> Dict[str, int]:
    n = C.c_int32()
    nnz = C.c_int64()
    nf = C.c_int64()
    s = _lib.mpap_roadmap_info(rm.handle, int(env), C.byref(n), C.byref(nnz), C.byref(nf))
    if s != MPAP_OK:
        raise MpapError(s, "mpap_roadmap_info")
    return {"n": n.value, "nnz": nnz.value, "nnz_free": nf.value}


def mpap_roadmap_export(rm: Roadmap, env: int = 0) -> Dict[str, np.ndarray]:
    info = mpap_roadmap_info(rm, env)
    n, nnz = info["n"], info["nnz"]
    row_ptr = np.zeros(n + 1, np.int32)
    dc = np.zeros(max(nnz, 1), np.uint32)
    w = np.zeros(max(nnz, 1), np.float32)
    s = np.zeros(max(nnz, 1), np.float32)
    c = np.zeros(max(nnz, 1), np.float32)
    st = _lib.mpap_roadmap_export(rm.handle, int(env), row_ptr.ctypes.data_as(_i32p), dc.ctypes.data, w.ctypes.data,
                                  s.ctypes.data, c.ctypes.data)
    if st != MPAP_OK:
        raise MpapError(st, "mpap_roadmap_export")
    return {"n": n, "row_ptr": row_ptr, "dst": (dc[:nnz] & 0x7FFFFFFF).astype(np.int32),
            "coll": (dc[:nnz] >> 31).astype(np.uint8), "w": w[:nnz], "s": s[:nnz], "c": c[:nnz]}


def mpap_roadmap_export_peaks(rm: Roadmap, env: int = 0):
    """Per-edge prefix maxima (S, C) of env's edges (f32 arrays [nnz])."""
    nnz = mpap_roadmap_info(rm, env)["nnz"]
    S = np.zeros(max(nnz, 1), np.float32)
    Cc = np.zeros(max(nnz, 1), np.float32)
    st = _lib.mpap_roadmap_export_peaks(rm.handle, int(env), S.ctypes.data, Cc.ctypes.data)
    if st != MPAP_OK:
        raise MpapError(st, "mpap_roadmap_export_peaks")
    return S[:nnz], Cc[:nnz]


def mpap_roadmap_set_peaks(rm: Roadmap, S, Cp) -> None:
    Sa = np.ascontiguousarray(S, dtype=np.float32)
    Ca = np.ascontiguousarray(Cp, dtype=np.float32)
    if Sa.size == 0:
        Sa, Ca = np.zeros(1, np.float32), np.zeros(1, np.float32)
    st = _lib.mpap_roadmap_set_peaks(rm.handle, Sa.ctypes.data, Ca.ctypes.data)
    if st != MPAP_OK:
        raise MpapError(st, "mpap_roadmap_set_peaks")


def mpap_roadmap_update(rm: Roadmap, env: int, obstacles, features, stream=None) -> int:
    """NEXT-1: replace env's obstacles [O, 2d] and features [F, d] (numpy or
    CUDA tensors) and re-evaluate only the affected edges; returns how many."""
    dev = _is_cuda_tensor(obstacles) or _is_cuda_tensor(features)
    mem = MPAP_MEM_DEVICE if dev else MPAP_MEM_HOST
    op, k1 = _ptr(obstacles, np.float64)
    fp, k2 = _ptr(features, np.float64)
    n = C.c_int64()
    st = _stream(stream)
    s = _lib.mpap_roadmap_update(rm.handle, int(env), op, int(obstacles.shape[0]), fp, int(features.shape[0]), mem,
                                 C.c_void_p(st) if st else None, C.byref(n))
    del k1, k2
    if s != MPAP_OK:
        raise MpapError(s, "mpap_roadmap_update")
    return int(n.value)


def mpap_launch_count() -> int:
    return int(_lib.mpap_launch_count())


def mpap_status_str(s: int) -> str:
    return _lib.mpap_status_str(int(s)).decode()


def mpap_prof_enable(on: bool = True) -> None:
    _lib.mpap_prof_enable(1 if on else 0)


def mpap_prof_reset() -> None:
    _lib.mpap_prof_reset()


def mpap_prof_read(kernel: str) -> tuple:
    """(total_ms, launches) of one library kernel since the last reset."""
    ms = C.c_double()
    n = C.c_int64()
    _lib.mpap_prof_read(kernel.encode(), C.byref(ms), C.byref(n))
    return float(ms.value), int(n.value)


def mpap_roadmap_block_device(rm: Roadmap, counts, edges, stream=None) -> int:
    """Write rm's row block into CUDA tensors: counts int32 [rows], edges
    int32 [capacity, 4] (16-byte records).  Returns the record count."""
    nnz = C.c_int64()
    st = _stream(stream)
    s = _lib.mpap_roadmap_block_device(rm.handle, C.c_void_p(int(counts.data_ptr())),
                                       C.c_void_p(int(edges.data_ptr())), int(edges.shape[0]), C.byref(nnz),
                                       C.c_void_p(st) if st else None)
    if s != MPAP_OK:
        raise MpapError(s, "mpap_roadmap_block_device")
    return int(nnz.value)


def mpap_roadmap_assemble_device(positions, row_begin, counts, edges, r: float, stream=None) -> Roadmap:
    """Assemble gathered row blocks (CUDA tensors counts int32 [B, rows_max],
    edges int32 [B, nnz_max, 4]) into a search roadmap on the device."""
    pos = np.ascontiguousarray(positions, dtype=np.float64)
    rb = np.ascontiguousarray(row_begin, dtype=np.int32)
    out = C.c_void_p()
    st = _stream(stream)
    s = _lib.mpap_roadmap_assemble_device(pos.shape[0], pos.shape[1], pos.ctypes.data, len(rb) - 1,
                                          rb.ctypes.data_as(_i32p), C.c_void_p(int(counts.data_ptr())),
                                          int(counts.shape[1]), C.c_void_p(int(edges.data_ptr())),
                                          int(edges.shape[1]), float(r), C.c_void_p(st) if st else None,
                                          C.byref(out))
    if s != MPAP_OK:
        raise MpapError(s, "mpap_roadmap_assemble_device")
    return Roadmap(out.value)


SEARCH_TEAMS = {"grid": 0, "cluster": 1, "cta": 2}


def mpap_search_launches() -> Dict[str, int]:
    """Search launches so far per team kind (grid / cluster / cta)."""
    if not hasattr(_lib, "mpap_search_launches"):
        return {}
    return {k: int(_lib.mpap_search_launches(v)) for k, v in SEARCH_TEAMS.items()}


def mpap_prof_fp64_peak(kind: str = "dfma") -> tuple:
    """(ops/s, ms) of the FP64 issue-rate microbenchmark: kind dfma, dadd or dmul."""
    k = {"dfma": 0, "dadd": 1, "dmul": 2}[kind]
    ops = C.c_double()
    ms = C.c_double()
    s = _lib.mpap_prof_fp64_peak(k, C.byref(ops), C.byref(ms))
    if s != MPAP_OK:
        raise MpapError(s, "mpap_prof_fp64_peak")
    return float(ops.value), float(ms.value)


KERNELS = ("k_near", "k_scan", "k_collide", "k_heuristic", "k_fold", "k_search")
MC_KERNELS = ("k_mc_plan", "k_mc")


WORK_FIELDS = ["pairs", "prefilter_pass", "bisect_iters", "edges", "coll_segs", "coll_box_tests", "steps",
               "range_tests", "fov_tests", "occl_segs", "occl_box_tests", "mlp", "free_edges", "cull_tests"]


def mpap_roadmap_work(rm: Roadmap) -> dict:
    """Build work counters of a roadmap (counted by the kernels)."""
    a = (C.c_uint64 * 16)()
    s = _lib.mpap_roadmap_work(rm.handle, a, 16)
    if s != MPAP_OK:
        raise MpapError(s, "mpap_roadmap_work")
    return {k: int(a[i]) for i, k in enumerate(WORK_FIELDS)}


def make_mc_params(mc: Dict[str, Any]) -> mpap_mc_params:
    """mpap_mc_params from a dict with the struct's field names."""
    return mpap_mc_params(trials=int(mc["trials"]), pad=0, seed=int(mc["seed"]) & (2 ** 64 - 1),
                          **{k: float(mc[k]) for k in ("sigma_imu", "sigma_vis", "u_max", "k_p", "k_d", "p0_pos",
                                                       "p0_vel", "delta")})


def mpap_mc_verify_batch(rm: Roadmap, envs, paths, path_lens, mc: Dict[str, Any], trial0: int = 0,
                         per_trial: bool = True, stream=None):
    """Monte Carlo verification (Alg. 1 step 4) of n plans: returns
    (results [n] MC_RESULT_DTYPE, max_err [n, trials], max_dev [n, trials])."""
    P = len(envs)
    ea = np.ascontiguousarray(envs, dtype=np.int32)
    pa = np.ascontiguousarray(paths, dtype=np.int32).reshape(P, -1)
    la = np.ascontiguousarray(path_lens, dtype=np.int32)
    m = make_mc_params(mc)
    res = np.zeros(max(P, 1), dtype=MC_RESULT_DTYPE)
    me = np.zeros((P, m.trials)) if per_trial else None
    md = np.zeros((P, m.trials)) if per_trial else None
    st = _stream(stream)
    s = _lib.mpap_mc_verify_batch(rm.handle, P, C.c_void_p(ea.ctypes.data), C.c_void_p(pa.ctypes.data),
                                  int(pa.shape[1]) if P else 1, C.c_void_p(la.ctypes.data), C.byref(m), int(trial0),
                                  C.c_void_p(me.ctypes.data) if per_trial else None,
                                  C.c_void_p(md.ctypes.data) if per_trial else None, C.c_void_p(res.ctypes.data),
                                  C.c_void_p(st) if st else None)
    if s != MPAP_OK:
        raise MpapError(s, "mpap_mc_verify_batch")
    return res[:P], me, md


def mpap_mc_verify(rm: Roadmap, env: int, path, mc: Dict[str, Any], trial0: int = 0, stream=None) -> Dict[str, Any]:
    """Monte Carlo verification of one plan: p_hat = P(max |x_hat - x| >= delta)."""
    pa = np.ascontiguousarray(path, dtype=np.int32)
    m = make_mc_params(mc)
    res = np.zeros(1, dtype=MC_RESULT_DTYPE)
    me = np.zeros(m.trials)
    md = np.zeros(m.trials)
    st = _stream(stream)
    s = _lib.mpap_mc_verify(rm.handle, int(env), C.c_void_p(pa.ctypes.data), len(pa), C.byref(m), int(trial0),
                            C.c_void_p(me.ctypes.data), C.c_void_p(md.ctypes.data), C.c_void_p(res.ctypes.data),
                            C.c_void_p(st) if st else None)
    if s != MPAP_OK:
        raise MpapError(s, "mpap_mc_verify")
    r = res[0]
    return {"p_hat": float(r["p_hat"]), "exceed": int(r["exceed"]), "trials": int(r["trials"]),
            "steps": int(r["steps"]), "fixes": int(r["fixes"]), "max_err": me, "max_dev": md}


def mpap_roadmap_rows_evaluated(rm: Roadmap, env: int = 0) -> int:
    """Rows of env whose collision bits and heuristic summaries exist (lazy
    roadmaps evaluate rows on first expansion; eager ones: all n)."""
    v = C.c_int64()
    s = _lib.mpap_roadmap_rows_evaluated(rm.handle, int(env), C.byref(v))
    if s != MPAP_OK:
        raise MpapError(s, "mpap_roadmap_rows_evaluated")
    return int(v.value)
