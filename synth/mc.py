"""Inputs of the Monte Carlo verification workload (NEXT-4): small hand-placed
problems for the oracle's pins and the per-config MC constants.

No method arithmetic here: these are input arrays and constants.  The
tracking gains are configuration values (a standard LQR design for the
per-axis double integrator with Q = diag(16, 0), R = 1, i.e. k_p = 4,
k_d = sqrt(8); SPEC lqr_gain S:357-363 gives the closed form), passed to both
implementations as plain numbers.
"""
from __future__ import annotations

import math
from typing import Any, Dict, Optional, Sequence

import numpy as np

from .envs import Problem

DEFAULT_MC: Dict[str, Any] = {
    "trials": 1000,          # Table 1 reports 1000 MC trials per plan
    "seed": 20170507,
    "sigma_imu": 0.3,        # m/s^2 per axis ("simulated accelerometer with noise")
    "sigma_vis": 0.1,        # m per axis per feature ("relative position with noise")
    "u_max": 5.0,            # m/s^2 per axis
    "k_p": 4.0,
    "k_d": math.sqrt(8.0),
    "p0_pos": 1e-4,
    "p0_vel": 1e-4,
    "delta": 0.3,            # m, localisation error bound (Eq. 1); profiles/r01/mc_sweep_c5.json
}


def mc_params(**over) -> Dict[str, Any]:
    d = dict(DEFAULT_MC)
    d.update(over)
    return d


def line_problem(points: Sequence[Sequence[float]], features: Optional[np.ndarray] = None,
                 obstacles: Optional[np.ndarray] = None, heuristic: int = 0, dt: float = 0.02,
                 max_range: float = 100.0, fov_half_deg: float = 45.0, r: float = 50.0) -> Problem:
    """A 3D double-integrator problem whose samples are the given states
    (p3, v3, cos yaw, sin yaw); the plan 0 -> 1 -> ... visits them in order."""
    smp = np.array([list(p) for p in points], dtype=np.float64)
    assert smp.shape[1] == 8
    feats = np.zeros((0, 3)) if features is None else np.asarray(features, dtype=np.float64).reshape(-1, 3)
    obst = np.zeros((0, 6)) if obstacles is None else np.asarray(obstacles, dtype=np.float64).reshape(-1, 6)
    params = {"control_weight": 1.0, "nominal_speed": 1.0, "dt": dt, "collision_dt": 0.1, "n_f": 12.0,
              "fov_cos_half": math.cos(math.radians(fov_half_deg)), "max_range": max_range, "mlp_gain": 0.0,
              "v_ref": 1.0, "w_ref": 1.0}
    return Problem(name="mc_line", pos_dim=3, dynamics=1, has_heading=1, heuristic=heuristic,
                   ws_lo=np.array([-100.0, -100.0, -100.0]), ws_hi=np.array([100.0, 100.0, 100.0]),
                   samples=smp, obstacles=obst, features=feats, params=params, mlp=np.zeros(122), r=r, lam=0.5,
                   start=0, goal_lo=smp[-1, :3].copy(), goal_hi=smp[-1, :3].copy())
