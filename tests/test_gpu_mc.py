"""GPU parity of the Monte Carlo verification (NEXT-4; Alg. 1 step 4,
P:290-292; model P:310-321; readings R31-R36): libmpap.so (k_mc_plan + k_mc
through the C ABI) vs the CPU oracle on identical inputs and noise streams.

Bar: per-trial max localisation error and max deviation bit-exact (f64), the
exceedance count and p_hat identical, step and fix counts equal.
"""
import numpy as np
import pytest

from synth import line_problem, load_config, make_problem, mc_params

pytestmark = pytest.mark.gpu
EAST = (1.0, 0.0)


@pytest.fixture(scope="module")
def mp():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import build_ext
    build_ext.build()
    import paper_1705_02408_b200 as m
    import paper_1705_02408_b200.problem as pb
    m.pb = pb
    return m


def check(g, o, trials):
    assert g["exceed"] == o["exceed"]
    assert np.array_equal(g["max_err"][:trials].view(np.uint64), o["max_err"][:trials].view(np.uint64)), \
        (g["max_err"][:4], o["max_err"][:4])
    assert np.array_equal(g["max_dev"][:trials].view(np.uint64), o["max_dev"][:trials].view(np.uint64))


def line(features, obstacles=None, heuristic=0, **kw):
    pts = [(0.0, 0.0, 1.5, 0.0, 0.0, 0.0, *EAST), (2.0, 0.5, 1.5, 0.5, 0.0, 0.0, *EAST),
           (4.0, 0.0, 1.5, 0.0, 0.0, 0.0, 0.0, 1.0)]
    return line_problem(pts, features=features, obstacles=obstacles, heuristic=heuristic, **kw)


@pytest.mark.parametrize("heur", [0, 1, 2, 3])
def test_mc_line_parity(mp, orc, heur):
    feats = [[2.0, 3.0, 1.5], [1.0, -2.0, 1.0], [5.0, 0.5, 2.0], [-1.0, 0.0, 1.5], [3.0, 1.0, 4.0]]
    wall = [[1.5, 1.2, 0.0, 2.5, 1.4, 3.0]]
    prob = line(feats, wall, heuristic=heur, max_range=4.0)
    rm = mp.pb.build_problem(prob)
    mc = mc_params(trials=96, sigma_imu=0.4, sigma_vis=0.1, delta=0.05)
    for path in ([0, 1, 2], [0, 2], [2, 1, 0], [1]):
        g = mp.mpap_mc_verify(rm, 0, path, mc, trial0=7)
        o = orc.mc_verify(prob, path, mc, 7)
        check(g, o, 96)
        t = orc.mc_trial(prob, path, mc, 7)
        assert g["steps"] == t["steps"]
    rm.free()


def test_mc_invalid_plan(mp):
    prob = line([[2.0, 3.0, 1.5]], obstacles=[[0.9, -1.0, 0.0, 1.1, 1.0, 3.0]])   # blocks 0 -> 1
    rm = mp.pb.build_problem(prob)
    with pytest.raises(mp.MpapError):
        mp.mpap_mc_verify(rm, 0, [0, 1], mc_params(trials=4))
    res, _, _ = mp.mpap_mc_verify_batch(rm, [0, 0], [[0, 1], [2, 2]], [2, 1], mc_params(trials=4))
    assert res["status"][0] == mp.MPAP_ERR_INVALID_ARGUMENT and res["status"][1] == 0
    with pytest.raises(mp.MpapError):
        mp.mpap_mc_verify(rm, 0, [0, 9], mc_params(trials=4))       # node out of range
    with pytest.raises(mp.MpapError):
        mp.mpap_mc_verify(rm, 0, [0, 2], mc_params(trials=0))       # no trials
    rm.free()


def c3_small():
    cfg = load_config("c3")
    cfg["n_samples"] = 400
    return make_problem(cfg)


def test_mc_c3_plan_parity(mp, orc):
    prob = c3_small()
    rm = mp.pb.build_problem(prob)
    mc = mc_params(trials=48)
    for beta in (float("inf"), 6.0):
        r = mp.pb.search_problem(rm, prob, beta)
        if r["status"] != 0:
            continue
        g = mp.mpap_mc_verify(rm, 0, r["path"], mc)
        o = orc.mc_verify(prob, r["path"], mc)
        check(g, o, 48)
        assert g["fixes"] > 0
    rm.free()


def test_mc_c5_batch_parity(mp, orc):
    """C5 environments at full size in the bench's batched launch: the GPU
    batch over 8 plans x 256 trials; the oracle recomputes sampled trials of
    each plan one by one."""
    cfg = load_config("c5")
    probs = [make_problem(cfg, env_index=k) for k in range(8)]
    B = mp.pb.Batch(probs)
    rm = B.build()
    paths, res = B.search(rm, [float(cfg["betas"][1])] * len(probs))
    mc = mc_params(trials=256)
    ok, mres, me = B.mc_verify(rm, paths, res, mc, per_trial=True)
    assert ok.size > 0 and np.all(mres["status"] == 0)
    for i, e in enumerate(ok[:4]):
        path = paths[e][: res["path_len"][e]]
        for t in (0, 1, 255):
            o = orc.mc_trial(probs[e], path, mc, t)
            assert me[i, t] == o["max_err"], (e, t)
        assert mres["steps"][i] == orc.mc_trial(probs[e], path, mc, 0)["steps"]
    rm.free()


def test_refine_beta_mc_parity(mp, orc):
    """Alg. 1 line 4: bound grid -> plans -> MC certificate;
    the GPU's table (status, cost, p_hat per bound) and its certified bound
    equal the oracle's search + MC over the same grid."""
    prob = c3_small()
    rm = mp.pb.build_problem(prob)
    orm = orc.build_roadmap(prob)
    mc = mc_params(trials=64, delta=0.15)
    betas = [2.0, 3.0, 4.5, 6.0, float("inf")]
    alpha = 0.25
    g = mp.pb.refine_beta_mc(rm, prob, betas, mc, alpha)
    best = None
    for row, beta in zip(g["table"], betas):
        o = orc.search(orm, prob, beta)
        assert row["status"] == o["status"], beta
        if o["status"] != 0:
            continue
        assert np.float32(row["cost"]) == o["cost"]
        om = orc.mc_verify(prob, o["path"], mc)
        assert row["p_hat"] == om["p_hat"], (beta, row["p_hat"], om["p_hat"])
        if om["p_hat"] <= alpha:
            best = beta
    assert g["certified"] == (best is not None)
    if best is not None:
        assert g["beta"] == best
    rm.free()


def test_mc_c2_velocity_fov_parity(mp, orc):
    """2D double integrator with the velocity-FOV heuristic (k_mc<2, 1>)."""
    cfg = load_config("c2")
    cfg["n_samples"] = 500
    prob = make_problem(cfg)
    rm = mp.pb.build_problem(prob)
    mc = mc_params(trials=64, sigma_imu=0.2, sigma_vis=0.05, delta=0.05)
    r = mp.pb.search_problem(rm, prob, float("inf"))
    assert r["status"] == 0
    g = mp.mpap_mc_verify(rm, 0, r["path"], mc)
    o = orc.mc_verify(prob, r["path"], mc)
    check(g, o, 64)
    rm.free()


def test_mc_kinematic_rejected(mp):
    cfg = load_config("c1")
    prob = make_problem(cfg)
    rm = mp.pb.build_problem(prob)
    with pytest.raises(mp.MpapError):
        mp.mpap_mc_verify(rm, 0, [0], mc_params(trials=4))
    rm.free()


def test_mc_c4_full_plan_sampled(mp, orc):
    """C4 at full size (n = 16 001, 200 boxes, 400 features): MC of the
    agnostic plan in one launch; sampled trials recomputed by the oracle."""
    cfg = load_config("c4")
    prob = make_problem(cfg)
    rm = mp.pb.build_problem(prob)
    r = mp.pb.search_problem(rm, prob, float("inf"))
    assert r["status"] == 0
    mc = mc_params(trials=128)
    g = mp.mpap_mc_verify(rm, 0, r["path"], mc)
    for t in (0, 77, 127):
        o = orc.mc_trial(prob, r["path"], mc, t)
        assert g["max_err"][t] == o["max_err"] and g["max_dev"][t] == o["max_dev"], t
    assert g["steps"] == orc.mc_trial(prob, r["path"], mc, 0)["steps"]
    rm.free()


def test_mc_large_trial_ids(mp, orc):
    """Trial ids beyond 32 bits (64-bit counter streams on both sides)."""
    prob = line([[2.0, 3.0, 1.5], [1.0, -2.0, 1.0]], heuristic=2, max_range=4.0)
    rm = mp.pb.build_problem(prob)
    mc = mc_params(trials=8, sigma_imu=0.4, sigma_vis=0.1, delta=0.05)
    t0 = (1 << 40) + 12345
    g = mp.mpap_mc_verify(rm, 0, [0, 1, 2], mc, trial0=t0)
    o = orc.mc_verify(prob, [0, 1, 2], mc, t0)
    check(g, o, 8)
    rm.free()
