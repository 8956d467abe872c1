"""Pins of the oracle's Monte Carlo verification (NEXT-4; Alg. 1 step 4,
P:180; simulation model of §4.1; readings R31-R36).

Each pin is fixed by mathematics, not by re-running the oracle's formulas:
* the noise generator has mean 0, variance 1 and support [-6, 6] (Irwin-Hall);
* zero noise: estimate == truth, tracking converges at first order in dt;
* IMU only: the estimation error is double-integrated white noise, whose
  variance after n steps is sigma^2 dt^4 n(n+1)(2n+1)/6 (closed form) -- the
  filter covariance must equal it and the empirical variance must match it;
* an exact fix (sigma_vis = 0) makes the error vanish after every update;
* the Kalman filter is consistent: empirical error variance == covariance;
* an occluding box removes every fix; delta = 0 gives p_hat = 1;
* streams are per trial (order independent).
"""
import math

import numpy as np
import pytest

from synth import line_problem, mc_params

EAST = (1.0, 0.0)


def straight(length=3.0, y=0.0, z=1.5):
    return [(0.0, y, z, 0.0, 0.0, 0.0, *EAST), (length, y, z, 0.0, 0.0, 0.0, *EAST)]


def test_normal_moments(orc):
    z = np.array([orc.mc_normal(11, t, i) for t in range(4) for i in range(10000)])
    assert abs(z.mean()) < 4.0 / math.sqrt(z.size)
    assert abs(z.var() - 1.0) < 0.03
    assert z.min() >= -6.0 and z.max() <= 6.0
    # different trials and seeds give different streams
    assert orc.mc_normal(11, 0, 0) != orc.mc_normal(11, 1, 0)
    assert orc.mc_normal(11, 0, 0) != orc.mc_normal(12, 0, 0)


def test_zero_noise_tracks_exactly(orc):
    prob = line_problem(straight(), features=[[1.5, 2.0, 1.5]])
    devs = []
    for dt in (0.02, 0.01, 0.005):
        prob.params["dt"] = dt
        r = orc.mc_trial(prob, [0, 1], mc_params(sigma_imu=0.0, sigma_vis=0.0), 0)
        assert r["max_err"] < 1e-12
        assert r["fixes"] == r["steps"]
        devs.append(r["max_dev"])
    # semi-implicit Euler with piecewise-constant feed-forward: first order in dt
    assert devs[0] < 1e-2
    assert 1.6 < devs[0] / devs[1] < 2.5 and 1.6 < devs[1] / devs[2] < 2.5


def test_imu_only_closed_form(orc):
    prob = line_problem(straight())
    sig = 0.5
    mc = mc_params(sigma_imu=sig, p0_pos=0.0, p0_vel=0.0)
    r0 = orc.mc_trial(prob, [0, 1], mc, 0)
    n = r0["steps"]
    assert r0["fixes"] == 0 and r0["draws"] == 3 * n
    # uniform step Dl on the single edge: recover it from the draws of one trial
    tau = orc.cost_di(prob.samples[0], prob.samples[1], 3, 1.0, prob.r)[1]
    dl = tau / n
    var = sig ** 2 * dl ** 4 * n * (n + 1) * (2 * n + 1) / 6.0
    assert r0["p11"] == pytest.approx(var, rel=1e-9)
    errs = np.array([orc.mc_trial(prob, [0, 1], mc, t)["err_final"] for t in range(1500)])
    emp = errs.var(axis=0)
    assert np.all(np.abs(emp / var - 1.0) < 0.12), (emp, var)


def test_exact_fix_zeroes_error(orc):
    prob = line_problem(straight(), features=[[1.5, 3.0, 1.5]])
    r = orc.mc_trial(prob, [0, 1], mc_params(sigma_imu=1.0, sigma_vis=0.0), 3)
    assert r["fixes"] == r["steps"] > 0
    assert r["max_err"] < 1e-9
    assert r["p11"] == 0.0


def test_kalman_consistency(orc):
    feats = [[1.0, 3.0, 1.5], [2.0, -3.0, 1.0], [1.5, 0.5, 4.0]]
    prob = line_problem(straight(), features=feats)
    mc = mc_params(sigma_imu=0.4, sigma_vis=0.05)
    tr = [orc.mc_trial(prob, [0, 1], mc, t) for t in range(1500)]
    assert all(t["fixes"] == t["steps"] for t in tr)
    assert all(t["draws"] == 3 * t["steps"] * 4 for t in tr)   # 3 IMU + 3 x 3 features per step
    emp = np.array([t["err_final"] for t in tr]).var(axis=0)
    assert np.all(np.abs(emp / tr[0]["p11"] - 1.0) < 0.12), (emp, tr[0]["p11"])


def test_occluder_blocks_fixes(orc):
    feat = [[1.5, 3.0, 1.5]]
    wall = [[-1.0, 1.0, 0.0, 4.0, 1.2, 3.0]]   # between the line y = 0 and the feature
    r_open = orc.mc_trial(line_problem(straight(), features=feat), [0, 1], mc_params(), 0)
    r_wall = orc.mc_trial(line_problem(straight(), features=feat, obstacles=wall), [0, 1], mc_params(), 0)
    assert r_open["fixes"] == r_open["steps"] and r_wall["fixes"] == 0
    # out of range: no fixes either
    r_far = orc.mc_trial(line_problem(straight(), features=feat, max_range=2.0), [0, 1], mc_params(), 0)
    assert r_far["fixes"] == 0


def test_fov_heading(orc):
    # heading east; a feature straight ahead is in view, one behind is not
    ahead = orc.mc_trial(line_problem(straight(), features=[[10.0, 0.0, 1.5]], heuristic=2), [0, 1],
                         mc_params(), 0)
    behind = orc.mc_trial(line_problem(straight(), features=[[-10.0, 0.0, 1.5]], heuristic=2), [0, 1],
                          mc_params(), 0)
    assert ahead["fixes"] == ahead["steps"] and behind["fixes"] == 0


def test_delta_and_order_independence(orc):
    prob = line_problem(straight(), features=[[1.5, 3.0, 1.5]])
    all10 = orc.mc_verify(prob, [0, 1], mc_params(delta=0.0), 0, 10)
    assert all10["exceed"] == 10 and all10["p_hat"] == 1.0
    none = orc.mc_verify(prob, [0, 1], mc_params(delta=1e9), 0, 10)
    assert none["exceed"] == 0
    part = orc.mc_verify(prob, [0, 1], mc_params(), 5, 3)
    full = orc.mc_verify(prob, [0, 1], mc_params(), 0, 10)
    assert np.array_equal(part["max_err"], full["max_err"][5:8])


def test_more_features_do_not_hurt(orc):
    few = [[1.5, 3.0, 1.5]]
    many = few + [[0.5, -3.0, 1.0], [2.5, 2.0, 2.5], [1.0, 1.0, 3.5]]
    mc = mc_params(sigma_imu=0.5, sigma_vis=0.2)
    a = orc.mc_verify(line_problem(straight(), features=few), [0, 1], mc, 0, 300)["max_err"]
    b = orc.mc_verify(line_problem(straight(), features=many), [0, 1], mc, 0, 300)["max_err"]
    assert np.median(b) < np.median(a)


def test_multi_edge_plan_and_invalid(orc):
    pts = [(0.0, 0.0, 1.5, 0.0, 0.0, 0.0, *EAST), (2.0, 0.5, 1.5, 0.5, 0.0, 0.0, *EAST),
           (4.0, 0.0, 1.5, 0.0, 0.0, 0.0, 0.0, 1.0)]
    prob = line_problem(pts, features=[[2.0, 3.0, 1.5]], heuristic=3)
    r = orc.mc_trial(prob, [0, 1, 2], mc_params(sigma_imu=0.0, sigma_vis=0.0), 0)
    assert r["max_err"] < 1e-12 and r["max_dev"] < 2e-2 and r["steps"] > 0
    one = orc.mc_trial(prob, [0], mc_params(), 0)          # start in goal: no motion
    assert one["steps"] == 0 and one["max_err"] == 0.0
    with pytest.raises(ValueError):                        # identical positions: no edge (R7)
        orc.mc_trial(line_problem([pts[0], pts[0]]), [0, 1], mc_params(), 0)
