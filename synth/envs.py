"""Seeded synthetic workloads C1-C5 (BASELINE.json ``configs``).

Each config JSON under ``configs/`` fixes a layout generator, its seed and the
frozen constants (r_n, lambda, beta).  ``make_problem`` turns it into the input
arrays both implementations consume:

* ``samples``  float64 [n, stride]  row = p[d] (+ v[d] if double integrator)
                                    (+ cos yaw, sin yaw if has_heading)
  Row 0 is x_init (Alg. 2 line 1).  Rows 1..n are Halton
  samples whose position is strictly outside every closed box (SampleFree,
  P:188).  If no sample position lies in the closed goal box, the
  goal-box centre is appended ("must include at least one from X_goal";
  SPEC S:149) - DESIGN.md reading R19.
* ``obstacles`` float64 [O, 2d]   lo[d], hi[d] (axis-aligned boxes)
* ``features``  float64 [F, d]    kept >= ``feature_clearance`` outside every
                                  box (reading R22)
* ``mlp``       float64 [122]     synthetic seeded weights of the 3-8-8-2 ReLU
                                  net (reading R12)

Yaw -> (cos, sin) is computed here once with numpy (reading N1), so neither
implementation evaluates a transcendental function.
"""
from __future__ import annotations

import json
import math
import os
from dataclasses import dataclass, field
from typing import Any, Dict, List, Optional

import numpy as np

from .halton import halton_points

CONFIG_DIR = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "configs")

DYNAMICS = {"kinematic": 0, "double_integrator": 1}
HEURISTICS = {"omni_count": 0, "fov_velocity_count": 1, "fov_heading_count": 2, "fov_heading_mlp": 3}
MLP_SIZE = 24 + 8 + 64 + 8 + 16 + 2  # W1[8x3] b1[8] W2[8x8] b2[8] W3[2x8] b3[2]


@dataclass
class Problem:
    """One environment + query, as plain arrays (no method arithmetic)."""
    name: str
    pos_dim: int
    dynamics: int
    has_heading: int
    heuristic: int
    ws_lo: np.ndarray
    ws_hi: np.ndarray
    samples: np.ndarray
    obstacles: np.ndarray
    features: np.ndarray
    params: Dict[str, float]
    mlp: np.ndarray
    r: float
    lam: float
    start: int
    goal_lo: np.ndarray
    goal_hi: np.ndarray
    betas: List[float] = field(default_factory=list)
    meta: Dict[str, Any] = field(default_factory=dict)

    @property
    def n(self) -> int:
        return int(self.samples.shape[0])

    @property
    def stride(self) -> int:
        return int(self.samples.shape[1])


def load_config(name_or_path: str) -> Dict[str, Any]:
    path = name_or_path
    if not os.path.exists(path):
        path = os.path.join(CONFIG_DIR, name_or_path + ".json")
    with open(path) as f:
        cfg = json.load(f)
    return cfg


# ----------------------------------------------------------------------------
# geometry helpers used ONLY for input generation (rejection of samples /
# features / furniture); these are not the method's collision primitive.
# ----------------------------------------------------------------------------

def _inside_any_box(pts: np.ndarray, boxes: np.ndarray, d: int, margin: float = 0.0) -> np.ndarray:
    """True where a point lies in some closed box grown by ``margin``."""
    if boxes.shape[0] == 0:
        return np.zeros(pts.shape[0], dtype=bool)
    lo = boxes[:, :d] - margin
    hi = boxes[:, d:2 * d] + margin
    p = pts[:, None, :d]
    inside = np.all((p >= lo[None]) & (p <= hi[None]), axis=2)
    return np.any(inside, axis=1)


def _boxes_overlap(a_lo, a_hi, b_lo, b_hi) -> bool:
    return bool(np.all(a_lo <= b_hi) and np.all(b_lo <= a_hi))


# ----------------------------------------------------------------------------
# layouts
# ----------------------------------------------------------------------------

def _layout_unit_square(cfg: Dict[str, Any], rng: np.random.Generator):
    """C1/C2: random boxes in a unit square, features concentrated in an inner
    region ("low-cost trajectories around the outside of the workspace,
    but with a feature distribution favoring the inside")."""
    d = 2
    start = np.array(cfg["start_pos"], dtype=np.float64)
    g_lo = np.array(cfg["goal_lo"], dtype=np.float64)
    g_hi = np.array(cfg["goal_hi"], dtype=np.float64)
    hw_lo, hw_hi = cfg["half_width"]
    c_lo, c_hi = cfg["centre_range"]
    boxes = []
    while len(boxes) < cfg["n_obstacles"]:
        c = rng.uniform(c_lo, c_hi, size=d)
        hw = rng.uniform(hw_lo, hw_hi, size=d)
        lo, hi = c - hw, c + hw
        if np.all(lo <= start) and np.all(start <= hi):
            continue
        if _boxes_overlap(lo, hi, g_lo, g_hi):
            continue
        boxes.append(np.concatenate([lo, hi]))
    boxes = np.array(boxes, dtype=np.float64).reshape(-1, 2 * d)
    feats = []
    n_inner = cfg["features_inner"]
    in_lo = np.array(cfg["inner_lo"], dtype=np.float64)
    in_hi = np.array(cfg["inner_hi"], dtype=np.float64)
    ws_lo = np.array(cfg["ws_lo"], dtype=np.float64)
    ws_hi = np.array(cfg["ws_hi"], dtype=np.float64)
    clear = cfg.get("feature_clearance", 1e-3)
    while len(feats) < cfg["n_features"]:
        if len(feats) < n_inner:
            f = rng.uniform(in_lo, in_hi)
        else:
            f = rng.uniform(ws_lo, ws_hi)
        if _inside_any_box(f[None], boxes, d, clear)[0]:
            continue
        feats.append(f)
    return boxes, np.array(feats, dtype=np.float64).reshape(-1, d)


def _wall_with_door(x0: float, thick: float, y0: float, y1: float, door_y: float,
                    door_w: float, door_h: float, z_hi: float) -> List[np.ndarray]:
    """Thin wall across a corridor (x in [x0, x0+thick], y in [y0, y1]) with a
    door gap y in [door_y, door_y+door_w], z in [0, door_h]."""
    out = []
    if door_y > y0:
        out.append([x0, y0, 0.0, x0 + thick, door_y, z_hi])
    if door_y + door_w < y1:
        out.append([x0, door_y + door_w, 0.0, x0 + thick, y1, z_hi])
    out.append([x0, door_y, door_h, x0 + thick, door_y + door_w, z_hi])
    return [np.array(b, dtype=np.float64) for b in out]


def _layout_building(cfg: Dict[str, Any], rng: np.random.Generator):
    """C3-C5: indoor building ("features ... favor the high-cost
    hallway, representing an incomplete mapping in the low-cost hallway").

    Horizontal spines split the floor into corridors; the direct corridor
    (y in [0, 4]) is crossed by thin walls with door gaps and is feature-poor;
    the others are longer detours and feature-rich.  Furniture boxes rest on
    the floor (the vehicle can fly over them)."""
    d = 3
    ws_lo = np.array(cfg["ws_lo"], dtype=np.float64)
    ws_hi = np.array(cfg["ws_hi"], dtype=np.float64)
    X, Y, Z = ws_hi - ws_lo
    start = np.array(cfg["start_pos"], dtype=np.float64)
    g_lo = np.array(cfg["goal_lo"], dtype=np.float64)
    g_hi = np.array(cfg["goal_hi"], dtype=np.float64)
    spines = cfg["spines"]            # list of [y_lo, y_hi]
    spine_x = cfg["spine_x"]          # [x_lo, x_hi]
    thick = cfg.get("wall_thickness", 0.2)
    fixed = []
    for (ylo, yhi) in spines:
        fixed.append(np.array([spine_x[0], ylo, 0.0, spine_x[1], yhi, Z], dtype=np.float64))
    # corridor partitions with doors: list of [x, y_lo, y_hi, door_w]
    door_regions = []
    for (x, ylo, yhi, door_w) in cfg["partitions"]:
        door_y = float(rng.uniform(ylo + 0.3, yhi - 0.3 - door_w))
        fixed += _wall_with_door(x, thick, ylo, yhi, door_y, door_w, cfg.get("door_height", 2.2), Z)
        door_regions.append((x - 0.8, x + thick + 0.8))
    boxes = list(fixed)
    keep_clear = [
        (start - 0.6, start + 0.6),
        (g_lo - 0.3, g_hi + 0.3),
    ]
    n_total = cfg["n_obstacles"]
    fs_lo, fs_hi = cfg["furniture_size"]
    fh_lo, fh_hi = cfg["furniture_height"]
    tries = 0
    while len(boxes) < n_total:
        tries += 1
        if tries > 100000:
            raise RuntimeError("furniture placement failed")
        size = rng.uniform(fs_lo, fs_hi, size=2)
        h = float(rng.uniform(fh_lo, fh_hi))
        c = rng.uniform(ws_lo[:2] + size / 2, ws_hi[:2] - size / 2)
        lo = np.array([c[0] - size[0] / 2, c[1] - size[1] / 2, 0.0])
        hi = np.array([c[0] + size[0] / 2, c[1] + size[1] / 2, h])
        if any(_boxes_overlap(lo, hi, a, b) for (a, b) in keep_clear):
            continue
        if any(lo[0] <= xr1 and hi[0] >= xr0 for (xr0, xr1) in door_regions):
            continue
        if any(_boxes_overlap(lo, hi, f[:3], f[3:]) for f in fixed):
            continue
        boxes.append(np.concatenate([lo, hi]))
    boxes = np.array(boxes, dtype=np.float64).reshape(-1, 2 * d)
    # features: a fraction in the "rich" y-bands, the rest anywhere
    rich = cfg["feature_rich_bands"]  # list of [y_lo, y_hi]
    frac = cfg["feature_rich_fraction"]
    n_f = cfg["n_features"]
    n_rich = int(round(frac * n_f))
    clear = cfg.get("feature_clearance", 0.05)
    feats = []
    tries = 0
    while len(feats) < n_f:
        tries += 1
        if tries > 1000000:
            raise RuntimeError("feature placement failed")
        if len(feats) < n_rich:
            band = rich[int(rng.integers(len(rich)))]
            f = np.array([rng.uniform(ws_lo[0] + 0.05, ws_hi[0] - 0.05),
                          rng.uniform(band[0] + 0.05, band[1] - 0.05),
                          rng.uniform(ws_lo[2] + 0.2, ws_hi[2] - 0.2)])
        else:
            f = rng.uniform(ws_lo + 0.05, ws_hi - 0.05)
        if _inside_any_box(f[None], boxes, d, clear)[0]:
            continue
        feats.append(f)
    return boxes, np.array(feats, dtype=np.float64).reshape(-1, d)


LAYOUTS = {"unit_square": _layout_unit_square, "building": _layout_building}


# ----------------------------------------------------------------------------

def _sample_free(cfg, boxes, d, dyn, has_heading, start_index):
    ws_lo = np.array(cfg["ws_lo"], dtype=np.float64)
    ws_hi = np.array(cfg["ws_hi"], dtype=np.float64)
    n = cfg["n_samples"]
    dims = d + (d if dyn == 1 else 0) + (1 if has_heading else 0)
    vmax = cfg.get("v_max", 0.0)
    rows = []
    got = 0
    idx = start_index
    chunk = max(64, 2 * n)
    while got < n:
        u = halton_points(idx, chunk, dims)
        idx += chunk
        pos = ws_lo + (ws_hi - ws_lo) * u[:, :d]
        ok = ~_inside_any_box(pos, boxes, d)
        u = u[ok]
        pos = pos[ok]
        cols = [pos]
        if dyn == 1:
            cols.append(vmax * (2.0 * u[:, d:2 * d] - 1.0))
        if has_heading:
            yaw = -math.pi + 2.0 * math.pi * u[:, -1]
            cols.append(np.stack([np.cos(yaw), np.sin(yaw)], axis=1))
        blk = np.concatenate(cols, axis=1)
        rows.append(blk[: n - got])
        got += min(n - got, blk.shape[0])
    return np.concatenate(rows, axis=0)


def make_problem(cfg: Dict[str, Any], env_index: Optional[int] = None) -> Problem:
    """Build the arrays of one environment+query from a config dict.

    ``env_index`` selects one environment of a batch config (C5): seed
    ``env_seed_base + env_index`` and Halton start ``1 + halton_stride*env_index``.
    """
    d = int(cfg["pos_dim"])
    dyn = DYNAMICS[cfg["dynamics"]]
    heur = HEURISTICS[cfg["heuristic"]]
    has_heading = 1 if cfg.get("heading", False) else 0
    if env_index is None:
        seed = int(cfg["env_seed"])
        hstart = int(cfg.get("halton_start", 1))
    else:
        seed = int(cfg["env_seed_base"]) + int(env_index)
        hstart = 1 + int(cfg.get("halton_stride", 0)) * int(env_index)
    rng = np.random.default_rng(seed)
    boxes, feats = LAYOUTS[cfg["layout"]](cfg, rng)
    samples = _sample_free(cfg, boxes, d, dyn, has_heading, hstart)
    # x_init as row 0 (zero velocity, heading +x)
    srow = list(cfg["start_pos"])
    if dyn == 1:
        srow += [0.0] * d
    if has_heading:
        srow += [1.0, 0.0]
    srow = np.array(srow, dtype=np.float64)[None]
    g_lo = np.array(cfg["goal_lo"], dtype=np.float64)
    g_hi = np.array(cfg["goal_hi"], dtype=np.float64)
    pos = samples[:, :d]
    in_goal = np.all((pos >= g_lo) & (pos <= g_hi), axis=1)
    rows = [srow, samples]
    appended = False
    if not np.any(in_goal):
        grow = list(0.5 * (g_lo + g_hi))
        if dyn == 1:
            grow += [0.0] * d
        if has_heading:
            grow += [1.0, 0.0]
        rows.append(np.array(grow, dtype=np.float64)[None])
        appended = True
    samples = np.ascontiguousarray(np.concatenate(rows, axis=0), dtype=np.float64)
    mlp = np.zeros(MLP_SIZE, dtype=np.float64)
    if heur == 3:
        wrng = np.random.default_rng(int(cfg.get("mlp_seed", 7)))
        mlp = wrng.normal(0.0, float(cfg.get("mlp_std", 0.5)), size=MLP_SIZE).astype(np.float64)
    fov = float(cfg.get("fov_half_angle_deg", 45.0))
    params = {
        "control_weight": float(cfg.get("control_weight", 1.0)),
        "nominal_speed": float(cfg.get("nominal_speed", 1.0)),
        "dt": float(cfg.get("dt", 0.02)),
        "collision_dt": float(cfg.get("collision_dt", 0.1)),
        "n_f": float(cfg.get("n_f", 12.0)),
        "fov_cos_half": float(np.cos(np.deg2rad(fov))),
        "max_range": float(cfg["max_range"]),
        "mlp_gain": float(cfg.get("mlp_gain", 0.25)),
        "v_ref": float(cfg.get("v_ref", 1.0)),
        "w_ref": float(cfg.get("w_ref", 1.0)),
    }
    ws_lo = np.zeros(3)
    ws_hi = np.zeros(3)
    ws_lo[:d] = cfg["ws_lo"]
    ws_hi[:d] = cfg["ws_hi"]
    betas = [float("inf") if (b is None or b == "inf") else float(b) for b in cfg.get("betas", ["inf"])]
    return Problem(
        name=cfg["name"] if env_index is None else f'{cfg["name"]}[{env_index}]',
        pos_dim=d, dynamics=dyn, has_heading=has_heading, heuristic=heur,
        ws_lo=ws_lo, ws_hi=ws_hi, samples=samples,
        obstacles=np.ascontiguousarray(boxes, dtype=np.float64),
        features=np.ascontiguousarray(feats, dtype=np.float64),
        params=params, mlp=mlp, r=float(cfg["r"]), lam=float(cfg.get("lambda", 0.5)),
        start=0, goal_lo=g_lo, goal_hi=g_hi, betas=betas,
        meta={"seed": seed, "halton_start": hstart, "goal_appended": appended},
    )
