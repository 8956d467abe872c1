"""CPU oracle of the MPAP hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The
product path (``paper_1705_02408_b200``) never imports it and fails loudly if
its CUDA library is missing.

The arithmetic lives in ``mpap_oracle.c`` (plain sequential C, compiled with
``-ffp-contract=off -fno-fast-math``); this module only marshals numpy arrays
through ctypes.  See the C file's header for the paper passages it follows.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from typing import Any, Dict, Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "mpap_oracle.c")
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

CFLAGS = ["-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared"]


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (no FMA contraction, no fast-math)."""
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC):
        tmp = _LIB_PATH + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


class OrcParams(C.Structure):
    _fields_ = [
        ("pos_dim", C.c_int32), ("dynamics", C.c_int32), ("has_heading", C.c_int32), ("heuristic", C.c_int32),
        ("ws_lo", C.c_double * 3), ("ws_hi", C.c_double * 3),
        ("control_weight", C.c_double), ("nominal_speed", C.c_double), ("dt", C.c_double),
        ("collision_dt", C.c_double), ("n_f", C.c_double), ("fov_cos_half", C.c_double),
        ("max_range", C.c_double), ("mlp", C.POINTER(C.c_double)), ("mlp_gain", C.c_double),
        ("v_ref", C.c_double), ("w_ref", C.c_double),
    ]


class OrcEnv(C.Structure):
    _fields_ = [
        ("samples", C.POINTER(C.c_double)), ("n", C.c_int32), ("stride", C.c_int32),
        ("obstacles", C.POINTER(C.c_double)), ("n_obstacles", C.c_int32),
        ("features", C.POINTER(C.c_double)), ("n_features", C.c_int32),
        ("r", C.c_double), ("use_prefilter", C.c_int32),
    ]


class OrcResult(C.Structure):
    _fields_ = [
        ("status", C.c_int32), ("path_len", C.c_int32), ("waves", C.c_int32), ("pad", C.c_int32),
        ("cost", C.c_float), ("h", C.c_float), ("h_peak", C.c_float), ("pad2", C.c_float),
        ("relaxations", C.c_int64), ("labels_inserted", C.c_int64),
    ]


class OrcMc(C.Structure):
    _fields_ = [("trials", C.c_int32), ("pad", C.c_int32), ("seed", C.c_uint64),
                ("sigma_imu", C.c_double), ("sigma_vis", C.c_double), ("u_max", C.c_double),
                ("k_p", C.c_double), ("k_d", C.c_double), ("p0_pos", C.c_double), ("p0_vel", C.c_double),
                ("delta", C.c_double)]


class OrcMcTrace(C.Structure):
    _fields_ = [("err_final", C.c_double * 3), ("p11", C.c_double), ("p12", C.c_double), ("p22", C.c_double),
                ("steps", C.c_int64), ("draws", C.c_int64), ("fixes", C.c_int64)]


MC_FIELDS = ["trials", "seed", "sigma_imu", "sigma_vis", "u_max", "k_p", "k_d", "p0_pos", "p0_vel", "delta"]


def _mc_struct(mc: Dict[str, Any]) -> "OrcMc":
    return OrcMc(trials=int(mc.get("trials", 0)), pad=0, seed=int(mc["seed"]) & (2 ** 64 - 1),
                 **{k: float(mc[k]) for k in MC_FIELDS[2:]})


WAVE_FIELDS = ["i", "group", "relax", "beta_pass", "inserted", "killed", "touched", "stair_sum"]


class OrcWave(C.Structure):
    _fields_ = [(f, C.c_int64) for f in WAVE_FIELDS] + [("e_rows", C.c_int64)]


def _ptr(a: np.ndarray, ct):
    return a.ctypes.data_as(C.POINTER(ct))


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_LIB_PATH)
        dp = C.POINTER(C.c_double)
        L.orc_seg_hits_box.argtypes = [dp, dp, dp, dp, C.c_int]
        L.orc_seg_hits_box.restype = C.c_int
        L.orc_cost_kinematic.argtypes = [dp, dp, C.c_int]
        L.orc_cost_kinematic.restype = C.c_double
        L.orc_cost_di.argtypes = [dp, dp, C.c_int, C.c_double, C.c_double, dp, dp]
        L.orc_cost_di.restype = C.c_int
        L.orc_collision.argtypes = [C.POINTER(OrcEnv), C.POINTER(OrcParams), C.c_int, C.c_int, C.c_double]
        L.orc_collision.restype = C.c_int
        L.orc_visible_count.argtypes = [C.POINTER(OrcEnv), C.POINTER(OrcParams), dp, dp]
        L.orc_visible_count.restype = C.c_int
        L.orc_edge_increments.argtypes = [C.POINTER(OrcEnv), C.POINTER(OrcParams), C.c_int, C.c_int,
                                          C.c_double, C.c_double, dp, C.c_int]
        L.orc_edge_increments.restype = C.c_int
        L.orc_mlp_out0.argtypes = [dp, C.c_double, C.c_double, C.c_double]
        L.orc_mlp_out0.restype = C.c_double
        L.orc_di_state.argtypes = [dp, dp, C.c_int, C.c_double, C.c_double, dp, dp]
        L.orc_di_state.restype = None
        L.orc_fold_summary.argtypes = [dp, C.c_int, dp, dp]
        L.orc_fold_summary.restype = None
        L.orc_fold_stepwise.argtypes = [C.c_double, dp, C.c_int]
        L.orc_fold_stepwise.restype = C.c_double
        L.orc_edge.argtypes = [C.POINTER(OrcEnv), C.POINTER(OrcParams), C.c_int, C.c_int,
                               dp, dp, C.POINTER(C.c_int), dp, dp]
        L.orc_edge.restype = C.c_int
        i32p, u8p, f32p = C.POINTER(C.c_int32), C.POINTER(C.c_uint8), C.POINTER(C.c_float)
        L.orc_build.argtypes = [C.POINTER(OrcEnv), C.POINTER(OrcParams), i32p, i32p, u8p, f32p, f32p, f32p,
                                dp, C.c_int64]
        L.orc_build.restype = C.c_int64
        L.orc_build_row.argtypes = [C.POINTER(OrcEnv), C.POINTER(OrcParams), C.c_int, i32p, u8p, f32p, f32p,
                                    f32p, C.c_int64]
        L.orc_build_row.restype = C.c_int64
        L.orc_search.argtypes = [C.c_int32, i32p, i32p, u8p, f32p, f32p, f32p, u8p, C.c_int32, C.c_double,
                                 C.c_double, C.c_double, i32p, C.c_int32, C.POINTER(OrcResult),
                                 C.POINTER(OrcWave), C.c_int32]
        L.orc_search.restype = C.c_int
        L.orc_search_ex.argtypes = L.orc_search.argtypes + [f32p, f32p, C.c_int32]
        L.orc_search_ex.restype = C.c_int
        L.orc_fold_peak.argtypes = [dp, C.c_int, dp, dp]
        L.orc_fold_peak.restype = None
        L.orc_fold_stepwise_peak.argtypes = [C.c_double, dp, C.c_int]
        L.orc_fold_stepwise_peak.restype = C.c_double
        L.orc_edge_peak.argtypes = [C.POINTER(OrcEnv), C.POINTER(OrcParams), C.c_int, C.c_int, dp, dp]
        L.orc_edge_peak.restype = C.c_int
        L.orc_build_peaks.argtypes = [C.POINTER(OrcEnv), C.POINTER(OrcParams), i32p, i32p, f32p, f32p]
        L.orc_build_peaks.restype = None
        L.orc_goal_mask.argtypes = [dp, C.c_int32, C.c_int32, C.c_int32, dp, dp, u8p]
        L.orc_goal_mask.restype = None
        L.orc_mc_normal.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64]
        L.orc_mc_normal.restype = C.c_double
        L.orc_mc_trial.argtypes = [C.POINTER(OrcEnv), C.POINTER(OrcParams), i32p, C.c_int32, C.POINTER(OrcMc),
                                   C.c_uint64, dp, dp, C.POINTER(OrcMcTrace)]
        L.orc_mc_trial.restype = C.c_int
        L.orc_mc_verify.argtypes = [C.POINTER(OrcEnv), C.POINTER(OrcParams), i32p, C.c_int32, C.POINTER(OrcMc),
                                    C.c_uint64, C.c_int32, dp, dp]
        L.orc_mc_verify.restype = C.c_int64
        _lib = L
    return _lib


class _Ctx:
    """Keeps numpy buffers alive while the C structs point at them."""

    def __init__(self, prob, use_prefilter: bool = True, r: Optional[float] = None):
        self.samples = np.ascontiguousarray(prob.samples, dtype=np.float64)
        self.obstacles = np.ascontiguousarray(prob.obstacles, dtype=np.float64).reshape(-1)
        if self.obstacles.size == 0:
            self.obstacles = np.zeros(1)
        self.features = np.ascontiguousarray(prob.features, dtype=np.float64).reshape(-1)
        if self.features.size == 0:
            self.features = np.zeros(1)
        self.mlp = np.ascontiguousarray(prob.mlp, dtype=np.float64)
        p = prob.params
        self.prm = OrcParams(
            pos_dim=prob.pos_dim, dynamics=prob.dynamics, has_heading=prob.has_heading, heuristic=prob.heuristic,
            ws_lo=(C.c_double * 3)(*[float(x) for x in prob.ws_lo]),
            ws_hi=(C.c_double * 3)(*[float(x) for x in prob.ws_hi]),
            control_weight=p["control_weight"], nominal_speed=p["nominal_speed"], dt=p["dt"],
            collision_dt=p["collision_dt"], n_f=p["n_f"], fov_cos_half=p["fov_cos_half"],
            max_range=p["max_range"], mlp=_ptr(self.mlp, C.c_double), mlp_gain=p["mlp_gain"],
            v_ref=p["v_ref"], w_ref=p["w_ref"],
        )
        self.env = OrcEnv(
            samples=_ptr(self.samples, C.c_double), n=self.samples.shape[0], stride=self.samples.shape[1],
            obstacles=_ptr(self.obstacles, C.c_double), n_obstacles=prob.obstacles.shape[0],
            features=_ptr(self.features, C.c_double), n_features=prob.features.shape[0],
            r=float(prob.r if r is None else r), use_prefilter=1 if use_prefilter else 0,
        )


# ---------------------------------------------------------------------------
# primitives (for pins)
# ---------------------------------------------------------------------------

def seg_hits_box(A, B, lo, hi) -> bool:
    d = len(A)
    a = [np.ascontiguousarray(x, dtype=np.float64) for x in (A, B, lo, hi)]
    return bool(lib().orc_seg_hits_box(*[_ptr(x, C.c_double) for x in a], d))


def cost_kinematic(pu, pv) -> float:
    a = np.ascontiguousarray(pu, dtype=np.float64)
    b = np.ascontiguousarray(pv, dtype=np.float64)
    return float(lib().orc_cost_kinematic(_ptr(a, C.c_double), _ptr(b, C.c_double), len(a)))


def cost_di(su, sv, d: int, ru: float, r: float):
    """(c*, tau*) of the double-integrator connection, or None (no local
    minimiser on (0, r])."""
    a = np.ascontiguousarray(su, dtype=np.float64)
    b = np.ascontiguousarray(sv, dtype=np.float64)
    c = C.c_double()
    t = C.c_double()
    ok = lib().orc_cost_di(_ptr(a, C.c_double), _ptr(b, C.c_double), d, ru, r, C.byref(c), C.byref(t))
    return (c.value, t.value) if ok else None


def visible_count(prob, x, hv) -> int:
    ctx = _Ctx(prob)
    xa = np.zeros(3)
    ha = np.zeros(3)
    xa[: len(x)] = x
    ha[: len(hv)] = hv
    return int(lib().orc_visible_count(C.byref(ctx.env), C.byref(ctx.prm), _ptr(xa, C.c_double), _ptr(ha, C.c_double)))


def edge(prob, u: int, v: int, use_prefilter: bool = True) -> Optional[Dict[str, Any]]:
    ctx = _Ctx(prob, use_prefilter)
    c64 = C.c_double()
    tau = C.c_double()
    coll = C.c_int()
    s64 = C.c_double()
    h64 = C.c_double()
    ok = lib().orc_edge(C.byref(ctx.env), C.byref(ctx.prm), u, v, C.byref(c64), C.byref(tau), C.byref(coll),
                        C.byref(s64), C.byref(h64))
    if not ok:
        return None
    return {"c64": c64.value, "tau": tau.value, "coll": coll.value, "s64": s64.value, "c_h64": h64.value,
            "w": np.float32(c64.value), "s": np.float32(s64.value), "c": np.float32(h64.value)}


def edge_increments(prob, u: int, v: int, c64: float, tau: float) -> np.ndarray:
    ctx = _Ctx(prob)
    K = lib().orc_edge_increments(C.byref(ctx.env), C.byref(ctx.prm), u, v, c64, tau, None, 0)
    out = np.zeros(max(K, 1))
    lib().orc_edge_increments(C.byref(ctx.env), C.byref(ctx.prm), u, v, c64, tau, _ptr(out, C.c_double), K)
    return out[:K]


def mlp_out0(weights, z) -> float:
    """First output of the 3-8-8-2 ReLU net (R12) at input z (3 values)."""
    w = np.ascontiguousarray(weights, dtype=np.float64)
    assert w.size == 122
    return float(lib().orc_mlp_out0(_ptr(w, C.c_double), float(z[0]), float(z[1]), float(z[2])))


def di_state(su, sv, d: int, tau: float, t: float):
    """(position, velocity) at time t on the double-integrator edge cubic (R7 step 6)."""
    a = np.ascontiguousarray(su, dtype=np.float64)
    b = np.ascontiguousarray(sv, dtype=np.float64)
    x = np.zeros(3)
    v = np.zeros(3)
    lib().orc_di_state(_ptr(a, C.c_double), _ptr(b, C.c_double), d, float(tau), float(t),
                       _ptr(x, C.c_double), _ptr(v, C.c_double))
    return x[:d].copy(), v[:d].copy()


def collision(prob, u: int, v: int, tau: float) -> bool:
    ctx = _Ctx(prob)
    return bool(lib().orc_collision(C.byref(ctx.env), C.byref(ctx.prm), u, v, tau))


def fold_summary(inc) -> tuple:
    a = np.ascontiguousarray(inc, dtype=np.float64)
    s = C.c_double()
    c = C.c_double()
    lib().orc_fold_summary(_ptr(a, C.c_double), len(a), C.byref(s), C.byref(c))
    return s.value, c.value


def fold_peak(inc) -> tuple:
    a = np.ascontiguousarray(inc, dtype=np.float64)
    S = C.c_double()
    Cc = C.c_double()
    lib().orc_fold_peak(_ptr(a, C.c_double), len(a), C.byref(S), C.byref(Cc))
    return S.value, Cc.value


def fold_stepwise_peak(h0: float, inc) -> float:
    a = np.ascontiguousarray(inc, dtype=np.float64)
    return float(lib().orc_fold_stepwise_peak(h0, _ptr(a, C.c_double), len(a)))


def build_peaks(prob, rm) -> tuple:
    """(S, C) f32 peak summaries of every edge of an oracle roadmap (NEXT-3)."""
    ctx = _Ctx(prob)
    nnz = len(rm["dst"])
    S = np.zeros(max(nnz, 1), np.float32)
    Cc = np.zeros(max(nnz, 1), np.float32)
    rp = np.ascontiguousarray(rm["row_ptr"], dtype=np.int32)
    dst = np.ascontiguousarray(rm["dst"] if nnz else np.zeros(1, np.int32), dtype=np.int32)
    lib().orc_build_peaks(C.byref(ctx.env), C.byref(ctx.prm), _ptr(rp, C.c_int32), _ptr(dst, C.c_int32),
                          _ptr(S, C.c_float), _ptr(Cc, C.c_float))
    return S[:nnz].copy(), Cc[:nnz].copy()


def fold_stepwise(h0: float, inc) -> float:
    a = np.ascontiguousarray(inc, dtype=np.float64)
    return float(lib().orc_fold_stepwise(h0, _ptr(a, C.c_double), len(a)))


# ---------------------------------------------------------------------------
# Alg. 2 + heuristic, Alg. 3
# ---------------------------------------------------------------------------

def build_roadmap(prob, use_prefilter: bool = True, r: Optional[float] = None) -> Dict[str, np.ndarray]:
    ctx = _Ctx(prob, use_prefilter, r)
    n = prob.samples.shape[0]
    cap = int(max(1024, n * 256))
    while True:
        row_ptr = np.zeros(n + 1, dtype=np.int32)
        dst = np.zeros(cap, dtype=np.int32)
        coll = np.zeros(cap, dtype=np.uint8)
        w = np.zeros(cap, dtype=np.float32)
        s = np.zeros(cap, dtype=np.float32)
        c = np.zeros(cap, dtype=np.float32)
        tau = np.zeros(cap, dtype=np.float64)
        nnz = lib().orc_build(C.byref(ctx.env), C.byref(ctx.prm), _ptr(row_ptr, C.c_int32), _ptr(dst, C.c_int32),
                              _ptr(coll, C.c_uint8), _ptr(w, C.c_float), _ptr(s, C.c_float), _ptr(c, C.c_float),
                              _ptr(tau, C.c_double), cap)
        if nnz <= cap:
            break
        cap = int(nnz)
    return {"n": n, "row_ptr": row_ptr, "dst": dst[:nnz].copy(), "coll": coll[:nnz].copy(), "w": w[:nnz].copy(),
            "s": s[:nnz].copy(), "c": c[:nnz].copy(), "tau": tau[:nnz].copy()}


def build_row(prob, u: int, use_prefilter: bool = True) -> Dict[str, np.ndarray]:
    ctx = _Ctx(prob, use_prefilter)
    n = prob.samples.shape[0]
    cap = n
    dst = np.zeros(cap, dtype=np.int32)
    coll = np.zeros(cap, dtype=np.uint8)
    w = np.zeros(cap, dtype=np.float32)
    s = np.zeros(cap, dtype=np.float32)
    c = np.zeros(cap, dtype=np.float32)
    k = lib().orc_build_row(C.byref(ctx.env), C.byref(ctx.prm), u, _ptr(dst, C.c_int32), _ptr(coll, C.c_uint8),
                            _ptr(w, C.c_float), _ptr(s, C.c_float), _ptr(c, C.c_float), cap)
    return {"dst": dst[:k].copy(), "coll": coll[:k].copy(), "w": w[:k].copy(), "s": s[:k].copy(), "c": c[:k].copy()}


def goal_mask(prob) -> np.ndarray:
    smp = np.ascontiguousarray(prob.samples, dtype=np.float64)
    lo = np.zeros(3)
    hi = np.zeros(3)
    lo[: prob.pos_dim] = prob.goal_lo
    hi[: prob.pos_dim] = prob.goal_hi
    out = np.zeros(smp.shape[0], dtype=np.uint8)
    lib().orc_goal_mask(_ptr(smp, C.c_double), smp.shape[0], smp.shape[1], prob.pos_dim, _ptr(lo, C.c_double),
                        _ptr(hi, C.c_double), _ptr(out, C.c_uint8))
    return out


STATUS = {0: "OK", 3: "NO_FEASIBLE_PLAN", 4: "BUFFER_TOO_SMALL", 5: "OUT_OF_MEMORY"}


def search_csr(n: int, row_ptr, dst, coll, w, s, c, goal, start: int, beta: float, lam: float, r: float,
               path_cap: int = 65536, waves_cap: int = 100000, S=None, Cp=None, forall_t: bool = False
               ) -> Dict[str, Any]:
    """Alg. 3 on an explicit CSR (hand-built graphs or an oracle roadmap).
    With forall_t, the cutoff applies to every step of an edge via the peak
    summaries (S, Cp) (NEXT-3)."""
    row_ptr = np.ascontiguousarray(row_ptr, dtype=np.int32)
    dst = np.ascontiguousarray(dst, dtype=np.int32)
    coll = np.ascontiguousarray(coll, dtype=np.uint8)
    w = np.ascontiguousarray(w, dtype=np.float32)
    s = np.ascontiguousarray(s, dtype=np.float32)
    c = np.ascontiguousarray(c, dtype=np.float32)
    goal = np.ascontiguousarray(goal, dtype=np.uint8)
    if forall_t:
        S = np.ascontiguousarray(S, dtype=np.float32)
        Cp = np.ascontiguousarray(Cp, dtype=np.float32)
    if dst.size == 0:  # keep valid pointers
        dst, coll, w, s, c = np.zeros(1, np.int32), np.zeros(1, np.uint8), np.zeros(1, np.float32), \
            np.zeros(1, np.float32), np.zeros(1, np.float32)
        if forall_t:
            S, Cp = np.zeros(1, np.float32), np.zeros(1, np.float32)
    if not forall_t:
        S = Cp = np.zeros(1, np.float32)
    path = np.zeros(path_cap, dtype=np.int32)
    res = OrcResult()
    waves = (OrcWave * waves_cap)()
    lib().orc_search_ex(n, _ptr(row_ptr, C.c_int32), _ptr(dst, C.c_int32), _ptr(coll, C.c_uint8),
                        _ptr(w, C.c_float), _ptr(s, C.c_float), _ptr(c, C.c_float), _ptr(goal, C.c_uint8), start,
                        beta, lam, r, _ptr(path, C.c_int32), path_cap, C.byref(res), waves, waves_cap,
                        _ptr(S, C.c_float), _ptr(Cp, C.c_float), 1 if forall_t else 0)
    nw = min(res.waves, waves_cap)
    wave_arr = np.array([[getattr(waves[k], f) for f in WAVE_FIELDS] for k in range(nw)], dtype=np.int64).reshape(-1, 8)
    return {
        "status": int(res.status), "status_str": STATUS.get(int(res.status), "?"),
        "path": path[: res.path_len].copy() if res.status == 0 else np.zeros(0, np.int32),
        "cost": np.float32(res.cost), "h": np.float32(res.h), "h_peak": np.float32(res.h_peak),
        "waves": int(res.waves), "relaxations": int(res.relaxations), "labels_inserted": int(res.labels_inserted),
        "wave_counters": wave_arr,
        # SURVEY §8(d) algorithmic-bytes counters: E_rows (distinct-head row
        # entries per wave), sum G, F_reads (= stair_sum), L_ins
        "e_rows": int(sum(waves[k].e_rows for k in range(nw))),
        "e_rows_per_wave": [int(waves[k].e_rows) for k in range(nw)],
    }


def search(rm: Dict[str, np.ndarray], prob, beta: float, lam: Optional[float] = None,
           r: Optional[float] = None, start: Optional[int] = None, forall_t: bool = False) -> Dict[str, Any]:
    S = Cp = None
    if forall_t:
        if "S" not in rm:
            rm["S"], rm["C"] = build_peaks(prob, rm)
        S, Cp = rm["S"], rm["C"]
    return search_csr(rm["n"], rm["row_ptr"], rm["dst"], rm["coll"], rm["w"], rm["s"], rm["c"], goal_mask(prob),
                      prob.start if start is None else start, beta, prob.lam if lam is None else lam,
                      prob.r if r is None else r, S=S, Cp=Cp, forall_t=forall_t)


# ---------------------------------------------------------------------------
# harness-level parallelism: independent rows of Alg. 2 on several processes
# (each process runs the unchanged sequential per-row oracle; the assembled
# CSR is identical to orc_build's -- checked in tests/test_oracle_build.py)
# ---------------------------------------------------------------------------

def _rows_worker(args):
    prob, lo, hi, use_prefilter = args
    out = []
    for u in range(lo, hi):
        out.append(build_row(prob, u, use_prefilter))
    return out


def build_roadmap_parallel(prob, procs: int = 0, use_prefilter: bool = True) -> Dict[str, np.ndarray]:
    import multiprocessing as mp
    n = prob.samples.shape[0]
    procs = procs or os.cpu_count() or 1
    if procs <= 1:
        return build_roadmap(prob, use_prefilter)
    nchunk = procs * 8
    bounds = np.linspace(0, n, nchunk + 1).astype(int)
    ctx = mp.get_context("fork")
    with ctx.Pool(procs) as pool:
        parts = pool.map(_rows_worker, [(prob, int(bounds[k]), int(bounds[k + 1]), use_prefilter)
                                        for k in range(nchunk)])
    rows = [r for part in parts for r in part]
    row_ptr = np.zeros(n + 1, np.int32)
    row_ptr[1:] = np.cumsum([len(r["dst"]) for r in rows])
    cat = lambda k, dt: np.concatenate([r[k] for r in rows]).astype(dt) if rows else np.zeros(0, dt)
    return {"n": n, "row_ptr": row_ptr, "dst": cat("dst", np.int32), "coll": cat("coll", np.uint8),
            "w": cat("w", np.float32), "s": cat("s", np.float32), "c": cat("c", np.float32)}


# ---------------------------------------------------------------------------
# Monte Carlo verification (NEXT-4; Alg. 1 step 4, model P:310-321)
# ---------------------------------------------------------------------------

def mc_normal(seed: int, trial: int, idx: int) -> float:
    """Normal number `idx` of trial `trial` (counter-based, reading R33)."""
    return float(lib().orc_mc_normal(int(seed) & (2 ** 64 - 1), int(trial), int(idx)))


def mc_trial(prob, path, mc: Dict[str, Any], trial: int) -> Dict[str, Any]:
    """One closed-loop trial along `path`: max localisation error, max
    deviation from the nominal, and the pins' trace (final error, filter
    covariance, step/draw/fix counts)."""
    ctx = _Ctx(prob)
    p = np.ascontiguousarray(path, dtype=np.int32)
    m = _mc_struct(mc)
    e, dv = C.c_double(), C.c_double()
    tr = OrcMcTrace()
    s = lib().orc_mc_trial(C.byref(ctx.env), C.byref(ctx.prm), _ptr(p, C.c_int32), len(p), C.byref(m),
                           int(trial), C.byref(e), C.byref(dv), C.byref(tr))
    if s != 0:
        raise ValueError("invalid plan for Monte Carlo (not a double-integrator r-disc path)")
    return {"max_err": e.value, "max_dev": dv.value, "err_final": np.array(tr.err_final[:]),
            "p11": tr.p11, "p12": tr.p12, "p22": tr.p22, "steps": tr.steps, "draws": tr.draws,
            "fixes": tr.fixes}


def mc_verify(prob, path, mc: Dict[str, Any], trial0: int = 0, ntrials: Optional[int] = None) -> Dict[str, Any]:
    """Trials trial0 .. trial0+ntrials-1: per-trial max errors / deviations and
    the exceedance count (p_hat = exceed / trials)."""
    ctx = _Ctx(prob)
    p = np.ascontiguousarray(path, dtype=np.int32)
    m = _mc_struct(mc)
    nt = int(mc["trials"] if ntrials is None else ntrials)
    me = np.zeros(max(nt, 1))
    md = np.zeros(max(nt, 1))
    ex = lib().orc_mc_verify(C.byref(ctx.env), C.byref(ctx.prm), _ptr(p, C.c_int32), len(p), C.byref(m),
                             int(trial0), nt, _ptr(me, C.c_double), _ptr(md, C.c_double))
    if ex < 0:
        raise ValueError("invalid plan for Monte Carlo")
    return {"max_err": me[:nt], "max_dev": md[:nt], "exceed": int(ex), "p_hat": ex / nt if nt else 0.0}
