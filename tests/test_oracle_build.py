"""Pins of the oracle's build half (Alg. 2; heuristic P:323-328,
P:476-477) against closed forms, brute force, invariants and SPEC worked
examples -- never against a retyped copy of the oracle's own formula.

The double-integrator pins solve the two-point boundary value problem with a
4x4 linear solve and integrate the control effort numerically, a different
route from the oracle's expanded closed form c(tau) and quartic (R7)."""
import math

import numpy as np
import pytest

from synth import load_config, make_problem
from synth.envs import Problem


# ---------------------------------------------------------------------------
# geometry
# ---------------------------------------------------------------------------

def test_slab_spec_examples(orc):
    lo, hi = [0.0, 0.0, 0.0], [1.0, 1.0, 1.0]
    assert orc.seg_hits_box([-1, 0.5, 0.5], [2, 0.5, 0.5], lo, hi)          # S:63 through the centre
    assert not orc.seg_hits_box([-1, 2, 0.5], [2, 2, 0.5], lo, hi)          # S:64 separated by a plane
    assert orc.seg_hits_box([-1, 1.0, 0.5], [2, 1.0, 0.5], lo, hi)          # S:56 touching face = collision
    assert orc.seg_hits_box([0.5, 0.5, 0.5], [0.5, 0.5, 0.5], lo, hi)       # S:84 degenerate, inside
    assert not orc.seg_hits_box([1.5, 0.5, 0.5], [1.5, 0.5, 0.5], lo, hi)   # degenerate, outside
    assert orc.seg_hits_box([1.0, 1.0, 1.0], [1.0, 1.0, 1.0], lo, hi)       # corner point, closed box


def test_slab_vs_dense_sampling(orc):
    """200 random segments vs a random box set; exact slab result equals a
    1000-point dense sampling oracle except within 1e-9 of tangency."""
    rng = np.random.default_rng(11)
    boxes = []
    for _ in range(6):
        c = rng.uniform(0.2, 0.8, 3)
        hw = rng.uniform(0.05, 0.15, 3)
        boxes.append((c - hw, c + hw))
    t = np.linspace(0.0, 1.0, 1000)
    checked = 0
    for _ in range(200):
        A = rng.uniform(0, 1, 3)
        B = rng.uniform(0, 1, 3)
        pts = A[None] + t[:, None] * (B - A)[None]
        for lo, hi in boxes:
            exact = orc.seg_hits_box(A, B, lo, hi)
            # signed distance of the sampled points to the box (>0 outside)
            out = np.maximum(np.maximum(lo - pts, pts - hi), 0.0)
            dist = np.sqrt((out ** 2).sum(axis=1))
            inside = np.all((pts >= lo) & (pts <= hi), axis=1)
            depth = np.min(np.minimum(pts - lo, hi - pts), axis=1)
            if exact and not inside.any():
                # allowed only if the segment passes within sampling resolution
                assert dist.min() < 2e-3
            elif not exact:
                assert not inside.any()
            checked += 1
            if inside.any():
                assert exact
            if depth.max() > 1e-9 and inside.any():
                assert exact
    assert checked == 1200


def test_slab_symmetry(orc):
    rng = np.random.default_rng(3)
    for _ in range(500):
        A = rng.uniform(0, 1, 3)
        B = rng.uniform(0, 1, 3)
        c = rng.uniform(0.2, 0.8, 3)
        hw = rng.uniform(0.02, 0.2, 3)
        assert orc.seg_hits_box(A, B, c - hw, c + hw) == orc.seg_hits_box(B, A, c - hw, c + hw)


# ---------------------------------------------------------------------------
# Cost and Near
# ---------------------------------------------------------------------------

def test_kinematic_cost_examples(orc):
    assert orc.cost_kinematic([0, 0, 0], [3, 4, 0]) == 5.0
    assert orc.cost_kinematic([1, 2, 3], [1, 2, 3]) == 0.0


def _bvp_cost(p0, v0, p1, v1, tau, ru, nq=64):
    """Independent route: cubic coefficients from a linear solve of the
    boundary conditions, then Gauss-Legendre integration of 1 + r_u |u|^2."""
    d = len(p0)
    M = np.array([[1, 0, 0, 0], [0, 1, 0, 0], [1, tau, tau ** 2, tau ** 3], [0, 1, 2 * tau, 3 * tau ** 2]], float)
    xg, wg = np.polynomial.legendre.leggauss(nq)
    tt = 0.5 * tau * (xg + 1)
    energy = 0.0
    for j in range(d):
        a = np.linalg.solve(M, [p0[j], v0[j], p1[j], v1[j]])
        u = 2 * a[2] + 6 * a[3] * tt
        energy += 0.5 * tau * np.sum(wg * u * u)
    return tau + ru * energy


def _bvp_min(p0, v0, p1, v1, ru, tmax):
    from scipy.optimize import minimize_scalar
    grid = np.geomspace(1e-4, tmax, 4000)
    vals = np.array([_bvp_cost(p0, v0, p1, v1, t, ru, nq=8) for t in grid])
    k = int(np.argmin(vals))
    lo = grid[max(k - 1, 0)]
    hi = grid[min(k + 1, len(grid) - 1)]
    res = minimize_scalar(lambda t: _bvp_cost(p0, v0, p1, v1, t, ru), bounds=(lo, hi), method="bounded",
                          options={"xatol": 1e-12})
    return res.fun, res.x


def test_di_cost_rest_to_rest_closed_form(orc):
    """v0 = v1 = 0: c(tau) = tau + 12 r_u |a|^2 / tau^3 -> tau* = (36 r_u |a|^2)^(1/4),
    c* = 4 tau*/3 (calculus on the rest-to-rest minimum-energy cost)."""
    rng = np.random.default_rng(5)
    for _ in range(50):
        d = int(rng.integers(2, 4))
        p0 = rng.uniform(-2, 2, d)
        p1 = rng.uniform(-2, 2, d)
        ru = float(rng.uniform(0.2, 3.0))
        aa = float(np.sum((p1 - p0) ** 2))
        tau_star = (36.0 * ru * aa) ** 0.25
        su = np.concatenate([p0, np.zeros(d)])
        sv = np.concatenate([p1, np.zeros(d)])
        out = orc.cost_di(su, sv, d, ru, 10.0 * tau_star + 1.0)
        assert out is not None
        c, t = out
        assert abs(t - tau_star) <= 1e-9 * tau_star
        assert abs(c - 4.0 * tau_star / 3.0) <= 1e-12 * c


def test_di_cost_time_reversal(orc):
    """Cost((p0,v0),(p1,v1)) = Cost((p1,-v1),(p0,-v0)) (time reversal of the
    double integrator; same vv, av, aa)."""
    rng = np.random.default_rng(6)
    for _ in range(200):
        d = 3
        p0, p1 = rng.uniform(-1, 1, d), rng.uniform(-1, 1, d)
        v0, v1 = rng.uniform(-1, 1, d), rng.uniform(-1, 1, d)
        a = orc.cost_di(np.r_[p0, v0], np.r_[p1, v1], d, 1.0, 20.0)
        b = orc.cost_di(np.r_[p1, -v1], np.r_[p0, -v0], d, 1.0, 20.0)
        assert (a is None) == (b is None)
        if a is not None:
            assert abs(a[0] - b[0]) <= 1e-14 * a[0]


def test_di_cost_vs_bvp_minimisation(orc):
    """Random pairs: the oracle's (c*, tau*) equals a numerical minimisation of
    the BVP cost over tau (independent route), to the minimiser's accuracy."""
    rng = np.random.default_rng(7)
    n_checked = 0
    for _ in range(40):
        d = int(rng.integers(2, 4))
        p0, p1 = rng.uniform(-1, 1, d), rng.uniform(-1, 1, d)
        v0, v1 = rng.uniform(-0.8, 0.8, d), rng.uniform(-0.8, 0.8, d)
        ru = float(rng.uniform(0.5, 2.0))
        r = 50.0
        out = orc.cost_di(np.r_[p0, v0], np.r_[p1, v1], d, ru, r)
        ref_c, ref_t = _bvp_min(p0, v0, p1, v1, ru, r)
        assert out is not None
        c, t = out
        assert abs(c - ref_c) <= 1e-7 * ref_c, (c, ref_c)
        # the value at the oracle's tau agrees with the BVP integral
        assert abs(_bvp_cost(p0, v0, p1, v1, t, ru) - c) <= 1e-10 * c
        n_checked += 1
    assert n_checked == 40


def _tiny_problem(name, n=None, r=None, **over):
    cfg = load_config(name)
    if n is not None:
        cfg["n_samples"] = n
    if r is not None:
        cfg["r"] = r
    cfg.update(over)
    return make_problem(cfg)


@pytest.mark.parametrize("name,n", [("c1", 120), ("c2", 150), ("c3", 120)])
def test_prefilter_is_bit_exact(orc, name, n):
    """SURVEY §8(c) Near pin: the conservative prefilter never changes the
    roadmap (all-pairs scan without it is bit-identical)."""
    p = _tiny_problem(name, n=n)
    a = orc.build_roadmap(p, use_prefilter=True)
    b = orc.build_roadmap(p, use_prefilter=False)
    for k in ("row_ptr", "dst", "coll", "w", "s", "c"):
        assert np.array_equal(a[k], b[k]), k


def test_near_monotone_in_r(orc):
    """increasing r_n yields a superset of edges."""
    p1 = _tiny_problem("c2", n=150, r=1.0)
    p2 = _tiny_problem("c2", n=150, r=1.3)
    a = orc.build_roadmap(p1)
    b = orc.build_roadmap(p2)
    for u in range(p1.n):
        sa = set(a["dst"][a["row_ptr"][u]:a["row_ptr"][u + 1]].tolist())
        sb = set(b["dst"][b["row_ptr"][u]:b["row_ptr"][u + 1]].tolist())
        assert sa <= sb


def test_kinematic_roadmap_symmetric_and_strict(orc):
    """Euclidean rows come out symmetric (R6) and every edge has w < r."""
    p = _tiny_problem("c1", n=200)
    rm = orc.build_roadmap(p)
    E = set()
    for u in range(p.n):
        for e in range(rm["row_ptr"][u], rm["row_ptr"][u + 1]):
            E.add((u, int(rm["dst"][e])))
            assert rm["dst"][e] != u
    assert all((v, u) in E for (u, v) in E)
    assert np.all(rm["w"].astype(np.float64) <= p.r)
    # brute-force adjacency from numpy distances
    pos = p.samples[:, :2]
    D = np.sqrt(((pos[:, None, :] - pos[None, :, :]) ** 2).sum(-1))
    for u in range(p.n):
        want = [v for v in range(p.n) if v != u and D[u, v] < p.r and abs(D[u, v] - p.r) > 1e-12]
        got = set(rm["dst"][rm["row_ptr"][u]:rm["row_ptr"][u + 1]].tolist())
        assert set(want) <= got and len(got) - len(want) <= 1


def test_kinematic_collision_vs_dense_sampling(orc):
    p = _tiny_problem("c1", n=200)
    rm = orc.build_roadmap(p)
    t = np.linspace(0, 1, 1000)
    pos = p.samples[:, :2]
    for u in range(0, p.n, 7):
        for e in range(rm["row_ptr"][u], rm["row_ptr"][u + 1]):
            v = rm["dst"][e]
            pts = pos[u][None] + t[:, None] * (pos[v] - pos[u])[None]
            hit = False
            near = False
            for b in p.obstacles:
                lo, hi = b[:2], b[2:]
                inside = np.all((pts >= lo) & (pts <= hi), axis=1)
                hit |= bool(inside.any())
                out = np.maximum(np.maximum(lo - pts, pts - hi), 0.0)
                near |= bool(np.sqrt((out ** 2).sum(1)).min() < 1e-3)
            if not near:
                assert bool(rm["coll"][e]) == hit


def test_di_stored_cost_equals_bvp_integral_at_tau(orc):
    """The stored w of every sampled double-integrator edge equals the BVP
    integral J(tau) = int (1 + r_u |u|^2) dt of the cubic through the boundary
    states at the oracle's tau (R7).  (The polyline vertices themselves are
    pinned against an independent linear solve in
    tests/test_oracle_pins.py::test_di_polyline_vertices_on_linear_solve_cubic.)"""
    p = _tiny_problem("c3", n=150)
    rm = orc.build_roadmap(p)
    d = 3
    rows = p.samples
    checked = 0
    for u in range(0, p.n, 5):
        for e in range(rm["row_ptr"][u], rm["row_ptr"][u + 1]):
            v = int(rm["dst"][e])
            tau = rm["tau"][e]
            c_bvp = _bvp_cost(rows[u, :d], rows[u, d:2 * d], rows[v, :d], rows[v, d:2 * d], tau, 1.0)
            assert abs(c_bvp - float(rm["w"][e])) <= 2e-7 * c_bvp
            checked += 1
    assert checked > 50


# ---------------------------------------------------------------------------
# heuristic and its tropical summary (R10)
# ---------------------------------------------------------------------------

def test_increment_examples(orc):
    """k = n_f visible -> 0; k = 0 -> dt; k = n_f/2 -> dt/2."""
    # one edge along +x, features placed so that exactly k are visible at every step
    def prob(k):
        feats = np.array([[0.5, 5.0 + 0.01 * i] for i in range(k)] + [[50.0, 50.0]], float).reshape(-1, 2)
        samples = np.array([[0.0, 0.0], [0.1, 0.0]])
        return Problem(name="t", pos_dim=2, dynamics=0, has_heading=0, heuristic=0,
                       ws_lo=np.array([-100., -100, 0]), ws_hi=np.array([100., 100, 0]), samples=samples,
                       obstacles=np.zeros((0, 4)), features=feats,
                       params=dict(control_weight=1.0, nominal_speed=1.0, dt=0.025, collision_dt=0.1, n_f=12.0,
                                   fov_cos_half=0.7, max_range=10.0, mlp_gain=0.0, v_ref=1.0, w_ref=1.0),
                       mlp=np.zeros(122), r=1.0, lam=0.5, start=0, goal_lo=np.zeros(2), goal_hi=np.zeros(2))
    for k, want in [(12, 0.0), (0, 0.025), (6, 0.0125)]:
        p = prob(k)
        inc = orc.edge_increments(p, 0, 1, 0.1, 0.1)
        assert len(inc) == 4                       # K = ceil(0.1/0.025)
        assert np.all(inc == want), (k, inc)


def test_fold_spec_examples(orc):
    # h0 = 0, [0.1]*3 -> 0.3 ; h0 = 0.05, [-0.1, 0.1] -> 0.1
    assert abs(orc.fold_stepwise(0.0, [0.1, 0.1, 0.1]) - 0.3) < 1e-15
    assert orc.fold_stepwise(0.05, [-0.1, 0.1]) == 0.1
    s, c = orc.fold_summary([-0.1, 0.1])
    assert max(c, 0.05 + s) == 0.1


def test_tropical_summary_equals_stepwise_fold(orc):
    """R10: h -> max(c, h + s) equals the stepwise clamp fold for every h0 >= 0;
    bit-exact for dyadic increments (all sums exact), within 1e-12 otherwise."""
    rng = np.random.default_rng(1)
    for _ in range(300):
        K = int(rng.integers(1, 60))
        inc = rng.integers(-64, 65, K) / 1024.0         # dyadic
        s, c = orc.fold_summary(inc)
        for h0 in [0.0, 0.015625, 0.25, 1.0, float(rng.integers(0, 200)) / 256.0]:
            assert max(c, h0 + s) == orc.fold_stepwise(h0, inc)
        inc2 = rng.uniform(-0.05, 0.05, K)
        s2, c2 = orc.fold_summary(inc2)
        for h0 in [0.0, 0.01, 0.3]:
            assert abs(max(c2, h0 + s2) - orc.fold_stepwise(h0, inc2)) < 1e-12


def test_fold_invariants(orc):
    """fold >= 0; <= h0 + sum(max(inc,0)); exactly additive when all
    increments are >= 0."""
    rng = np.random.default_rng(2)
    for _ in range(200):
        inc = rng.uniform(-0.1, 0.1, int(rng.integers(1, 40)))
        h0 = float(rng.uniform(0, 0.5))
        h = orc.fold_stepwise(h0, inc)
        assert h >= 0 and h <= h0 + np.maximum(inc, 0).sum() + 1e-12
        pos = np.abs(inc)
        assert abs(orc.fold_stepwise(h0, pos) - (h0 + pos.sum())) < 1e-12


def _vis_problem(obstacles=None, fov_cos=math.cos(math.pi / 4), rng_=10.0):
    feats = np.array([[1.0, 0.0, 0.0], [-1.0, 0.0, 0.0]])
    return Problem(name="v", pos_dim=3, dynamics=0, has_heading=1, heuristic=2,
                   ws_lo=np.array([-10., -10, -10]), ws_hi=np.array([10., 10, 10]),
                   samples=np.zeros((1, 5)), obstacles=(np.zeros((0, 6)) if obstacles is None else obstacles),
                   features=feats,
                   params=dict(control_weight=1.0, nominal_speed=1.0, dt=0.02, collision_dt=0.1, n_f=12.0,
                               fov_cos_half=fov_cos, max_range=rng_, mlp_gain=0.0, v_ref=1.0, w_ref=1.0),
                   mlp=np.zeros(122), r=1.0, lam=0.5, start=0, goal_lo=np.zeros(3), goal_hi=np.zeros(3))


def test_visibility_spec_examples(orc):
    """feature 1 m ahead visible; directly behind not; occluded not."""
    p = _vis_problem()
    assert orc.visible_count(p, [0, 0, 0], [1, 0, 0]) == 1        # the +x feature only
    assert orc.visible_count(p, [0, 0, 0], [0, 1, 0]) == 0        # both at 90 deg > 45 deg
    occl = np.array([[0.4, -0.1, -0.1, 0.6, 0.1, 0.1]])
    assert orc.visible_count(_vis_problem(occl), [0, 0, 0], [1, 0, 0]) == 0
    assert orc.visible_count(_vis_problem(rng_=0.5), [0, 0, 0], [1, 0, 0]) == 0   # out of range


def test_visibility_monotone(orc):
    """enlarging FOV or range never removes a feature; removing an
    obstacle never shrinks the visible set."""
    rng = np.random.default_rng(4)
    for _ in range(100):
        feats = rng.uniform(-3, 3, (20, 3))
        obst = []
        for _ in range(4):
            c = rng.uniform(-2, 2, 3)
            hw = rng.uniform(0.1, 0.5, 3)
            obst.append(np.r_[c - hw, c + hw])
        obst = np.array(obst)
        x = rng.uniform(-3, 3, 3)
        hv = rng.normal(size=3)
        base = _vis_problem(obst, 0.7, 2.0)
        base.features = feats
        k0 = orc.visible_count(base, x, hv)
        wide = _vis_problem(obst, 0.5, 2.0)
        wide.features = feats
        far = _vis_problem(obst, 0.7, 3.0)
        far.features = feats
        fewer = _vis_problem(obst[1:], 0.7, 2.0)
        fewer.features = feats
        assert orc.visible_count(wide, x, hv) >= k0
        assert orc.visible_count(far, x, hv) >= k0
        assert orc.visible_count(fewer, x, hv) >= k0


def test_mlp_zero_weights_reduce_to_count(orc):
    """R12 pin: with all-zero weights the learned-style increment equals the
    feature-count increment exactly, so (s, c) are bit-identical."""
    p3 = _tiny_problem("c3", n=80)
    p3.mlp = np.zeros(122)
    p2 = _tiny_problem("c3", n=80)
    p2.heuristic = 2
    a = orc.build_roadmap(p3)
    b = orc.build_roadmap(p2)
    for k in ("dst", "coll", "w", "s", "c"):
        assert np.array_equal(a[k], b[k])


def test_edge_without_features_in_range_costs_tau(orc):
    """Closed form: if no feature is ever visible, every increment is Delta and
    the clamp never fires, so s = c = K * Delta = tau (up to K roundings)."""
    p = _tiny_problem("c2", n=150)
    p.features = np.array([[100.0, 100.0]])
    rm = orc.build_roadmap(p)
    free = rm["coll"] == 0
    tau = rm["tau"][free]
    assert np.allclose(rm["s"][free], tau.astype(np.float32), rtol=1e-6)
    assert np.array_equal(rm["s"][free], rm["c"][free])
