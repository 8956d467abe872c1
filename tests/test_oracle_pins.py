"""Pins of the oracle functions that round 1 left unpinned (VERDICT r01,
"Parity unpinned"): the learned-style MLP (R12), the collision of
curved double-integrator edges (R8) and the FOV cone around the
interpolated heading (R9).  Each is checked against an independent
route -- exact rational arithmetic, an independent linear solve of the cubic
and dense sampling, angles from atan2 -- chosen so that a transposed weight
matrix, a swapped input, a reversed heading interpolation or a wrong polyline
vertex fails.  CPU only (-m "not gpu")."""
import math
from fractions import Fraction

import numpy as np
import pytest

from synth import load_config, make_problem
from synth.mc import line_problem


def _tiny(name, n, **over):
    cfg = load_config(name)
    cfg["n_samples"] = n
    cfg.update(over)
    return make_problem(cfg)


# ---------------------------------------------------------------------------
# (a) learned-style MLP, R12 / P:476-477: o = W3 relu(W2 relu(W1 z + b1) + b2) + b3
# ---------------------------------------------------------------------------

def _mlp_exact(w, z):
    """Forward pass in exact rational arithmetic (plain definition; weight
    layout W1[8x3] b1[8] W2[8x8] b2[8] W3[2x8] b3[2], row-major, R12) plus the
    same pass on absolute values (the forward error bound's scale)."""
    F = [Fraction(float(x)) for x in w]
    W1 = [[F[i * 3 + j] for j in range(3)] for i in range(8)]
    b1 = F[24:32]
    W2 = [[F[32 + i * 8 + j] for j in range(8)] for i in range(8)]
    b2 = F[96:104]
    W3 = [[F[104 + i * 8 + j] for j in range(8)] for i in range(2)]
    b3 = F[120:122]
    zf = [Fraction(float(x)) for x in z]
    h1 = [max(Fraction(0), b1[i] + sum(W1[i][j] * zf[j] for j in range(3))) for i in range(8)]
    h2 = [max(Fraction(0), b2[i] + sum(W2[i][j] * h1[j] for j in range(8))) for i in range(8)]
    o = b3[0] + sum(W3[0][j] * h2[j] for j in range(8))
    a1 = [abs(b1[i]) + sum(abs(W1[i][j] * zf[j]) for j in range(3)) for i in range(8)]
    a2 = [abs(b2[i]) + sum(abs(W2[i][j]) * a1[j] for j in range(8)) for i in range(8)]
    scale = abs(b3[0]) + sum(abs(W3[0][j]) * a2[j] for j in range(8))
    return float(o), float(scale)


def test_mlp_out0_vs_exact_forward_pass(orc):
    """Random weights and inputs: the oracle's fp64 fma chains equal the exact
    forward pass within the forward error bound 32 u * (|W3| (|W2| (|W1||z| +
    |b1|) + |b2|) + |b3|).  A transposed W1/W2, a swapped input or W3's second
    row instead of its first misses by O(1)."""
    rng = np.random.default_rng(17)
    u = 2.0 ** -53
    worst = 0.0
    for trial in range(200):
        w = rng.normal(0.0, 0.5, size=122)
        z = rng.uniform(-0.5, 2.0, size=3)
        got = orc.mlp_out0(w, z)
        want, scale = _mlp_exact(w, z)
        assert abs(got - want) <= 32 * u * scale, (trial, got, want)
        worst = max(worst, abs(got - want) / max(scale, 1e-300))
    # the net is not trivial on these inputs (outputs vary by O(1))
    outs = [orc.mlp_out0(rng.normal(0, 0.5, 122), rng.uniform(0, 1, 3)) for _ in range(20)]
    assert np.std(outs) > 0.1


def test_mlp_layout_mistakes_are_caught(orc):
    """The pin above is sensitive to the plausible layout mistakes."""
    rng = np.random.default_rng(3)
    w = rng.normal(0.0, 0.5, size=122)
    z = np.array([0.7, 0.3, 0.25])
    want, scale = _mlp_exact(w, z)
    wt = w.copy()
    wt[:24] = w[:24].reshape(3, 8).T.reshape(-1)                  # W1[i][j] read as w[j*8 + i]
    bad = [orc.mlp_out0(wt, z),                                   # W1 read column-major
           orc.mlp_out0(w, z[[1, 0, 2]]),                          # inputs swapped
           orc.mlp_out0(np.concatenate([w[:104], w[112:120], w[104:112], w[121:], w[120:121]]), z)]  # W3 row 1
    for b in bad:
        assert abs(b - want) > 1e3 * 32 * 2.0 ** -53 * scale


def _cubic_np(su, sv, d, tau):
    """Cubic p(t) = a0 + a1 t + a2 t^2 + a3 t^3 through (p0, v0) at 0 and
    (p1, v1) at tau, by an independent 4x4 linear solve per axis (R7 step 6)."""
    M = np.array([[1, 0, 0, 0], [0, 1, 0, 0], [1, tau, tau ** 2, tau ** 3], [0, 1, 2 * tau, 3 * tau ** 2]])
    return np.array([np.linalg.solve(M, [su[j], su[d + j], sv[j], sv[d + j]]) for j in range(d)])  # [d][4]


def _pos(A, t):
    t = np.asarray(t, dtype=np.float64)
    return A[:, 0][None] + np.outer(t, A[:, 1]) + np.outer(t ** 2, A[:, 2]) + np.outer(t ** 3, A[:, 3])


def _vel(A, t):
    t = np.asarray(t, dtype=np.float64)
    return A[:, 1][None] + np.outer(2 * t, A[:, 2]) + np.outer(3 * t ** 2, A[:, 3])


def test_mlp_increments_on_edges_vs_numpy_forward(orc):
    """R12 on whole edges of a C3-shaped roadmap with its seeded (non-zero)
    weights: inc_mlp - inc_count = Delta * gamma * out0(z) at every step, with
    z = (|v(t)|/v_ref, omega/w_ref, k_vis/n_f) computed independently (speed
    from the linear-solve cubic, omega from the headings, k_vis recovered from
    the count increments) and out0 by the exact forward pass."""
    p3 = _tiny("c3", 120)
    assert np.abs(p3.mlp).max() > 0 and p3.params["mlp_gain"] > 0
    p2 = _tiny("c3", 120)
    p2.heuristic = 2
    rm = orc.build_roadmap(p3)
    d = 3
    gam = p3.params["mlp_gain"]
    nf = p3.params["n_f"]
    checked = 0
    for u in range(0, p3.n, 9):
        for e in range(rm["row_ptr"][u], rm["row_ptr"][u + 1]):
            if rm["coll"][e]:
                continue
            v = int(rm["dst"][e])
            ed = orc.edge(p3, u, v)
            inc3 = orc.edge_increments(p3, u, v, ed["c64"], ed["tau"])
            inc2 = orc.edge_increments(p2, u, v, ed["c64"], ed["tau"])
            K = len(inc3)
            tau = ed["tau"]
            assert K == max(1, math.ceil(tau / p3.params["dt"])) and len(inc2) == K
            Dl = tau / K
            su, sv = p3.samples[u], p3.samples[v]
            A = _cubic_np(su, sv, d, tau)
            t = np.arange(K) * Dl
            speed = np.linalg.norm(_vel(A, t), axis=1)
            omega = math.hypot(sv[6] - su[6], sv[7] - su[7]) / tau
            kv = np.rint((Dl - inc2) * nf / Dl)
            assert np.allclose((Dl - inc2) * nf / Dl, kv, atol=1e-9)
            for k in range(0, K, 3):
                z = (speed[k] / p3.params["v_ref"], omega / p3.params["w_ref"], kv[k] / nf)
                want, scale = _mlp_exact(p3.mlp, z)
                got = (inc3[k] - inc2[k]) / (Dl * gam)
                assert abs(got - want) <= 1e-9 * (1.0 + scale), (u, v, k, got, want)
                checked += 1
    assert checked > 200


# ---------------------------------------------------------------------------
# (b) collision of curved double-integrator edges, R8 / P:190
# ---------------------------------------------------------------------------

def _box_depth_and_dist(pts, lo, hi):
    """Per point: depth inside the closed box (min distance to a face, < 0
    outside) and Euclidean distance to the box (0 inside)."""
    depth = np.minimum(pts - lo, hi - pts).min(axis=1)
    out = np.maximum(np.maximum(lo - pts, pts - hi), 0.0)
    return depth, np.sqrt((out ** 2).sum(1))


def _polyline_collision_np(prob, A, tau, dense=1000):
    """Independent R8: vertices P_k = p(k tau / Kc) of the linear-solve cubic,
    any vertex outside the workspace or any segment touching a closed box is a
    collision, decided by dense sampling (dense points per segment).  Returns
    (decision, certain): certain is False within 1e-6 m of a box / workspace
    face (tangency)."""
    d = prob.pos_dim
    Kc = max(1, math.ceil(tau / prob.params["collision_dt"]))
    V = _pos(A, np.arange(Kc + 1) * tau / Kc)
    lo_ws, hi_ws = np.asarray(prob.ws_lo[:d]), np.asarray(prob.ws_hi[:d])
    ws_depth = np.minimum(V - lo_ws, hi_ws - V).min()
    if ws_depth < -1e-6:
        return True, True
    certain = ws_depth > 1e-6
    s = np.linspace(0.0, 1.0, dense)
    pts = (V[:-1, None, :] + s[None, :, None] * (V[1:] - V[:-1])[:, None, :]).reshape(-1, d)
    blo, bhi = pts.min(0) - 1e-3, pts.max(0) + 1e-3
    hit = False
    for b in prob.obstacles:
        lo, hi = b[:d], b[d:]
        if np.any(lo > bhi) or np.any(hi < blo):
            continue
        depth, dist = _box_depth_and_dist(pts, lo, hi)
        if depth.max() > 1e-6:
            return True, True
        if depth.max() >= -1e-6 or dist.min() < 1e-3:
            certain = False      # grazing: the sampled decision is not certain
    return hit, certain


def test_di_collision_vs_dense_polyline_sampling(orc):
    """orc_collision on C3-shaped double-integrator roadmaps equals dense
    sampling (1000 points per segment) of the polyline through the
    independently solved cubic, plus the vertex workspace test, excluding
    near-tangent edges.  Both outcomes must be well represented."""
    n_hit = n_free = 0
    for seed in (3, 11):
        p = _tiny("c3", 400, env_seed=seed)
        rm = orc.build_roadmap(p)
        for u in range(0, p.n, 2):
            for e in range(rm["row_ptr"][u], rm["row_ptr"][u + 1]):
                v = int(rm["dst"][e])
                tau = float(rm["tau"][e])
                A = _cubic_np(p.samples[u], p.samples[v], 3, tau)
                want, certain = _polyline_collision_np(p, A, tau)
                if not certain:
                    continue
                assert bool(rm["coll"][e]) == want, (seed, u, v)
                n_hit += want
                n_free += not want
    assert n_hit >= 100 and n_free >= 300, (n_hit, n_free)


def test_di_collision_vs_dense_cubic_sampling(orc):
    """Away from the polyline's chord error the polyline decision is the cubic's:
    edges whose sampled cubic (1000 points per polyline segment) is either
    inside a box by more than the chord deviation or clear of every box by
    more than it agree with orc_collision."""
    p = _tiny("c3", 400, env_seed=5)
    rm = orc.build_roadmap(p)
    n = n_in = 0
    for u in range(0, p.n, 3):
        for e in range(rm["row_ptr"][u], rm["row_ptr"][u + 1]):
            v = int(rm["dst"][e])
            tau = float(rm["tau"][e])
            A = _cubic_np(p.samples[u], p.samples[v], 3, tau)
            Kc = max(1, math.ceil(tau / p.params["collision_dt"]))
            t = np.linspace(0.0, tau, 1000 * Kc + 1)
            pts = _pos(A, t)
            V = _pos(A, np.arange(Kc + 1) * tau / Kc)
            # chord deviation bound: distance of the cubic samples from the polyline
            seg = np.minimum((t * Kc / tau).astype(int), Kc - 1)
            s = t * Kc / tau - seg
            chord = V[seg] + s[:, None] * (V[seg + 1] - V[seg])
            dev = np.sqrt(((pts - chord) ** 2).sum(1)).max() + 1e-6
            inside = False
            clear = True
            blo, bhi = pts.min(0) - dev - 1e-3, pts.max(0) + dev + 1e-3
            for b in p.obstacles:
                if np.any(b[:3] > bhi) or np.any(b[3:] < blo):
                    continue
                depth, dist = _box_depth_and_dist(pts, b[:3], b[3:])
                if depth.max() > dev:
                    inside = True
                if dist.min() <= dev:
                    clear = False
            ws_clear = np.all(pts > p.ws_lo[:3] + dev) and np.all(pts < p.ws_hi[:3] - dev)
            if inside:
                assert rm["coll"][e] == 1, (u, v)
                n += 1
                n_in += 1
            elif clear and ws_clear:
                assert rm["coll"][e] == 0, (u, v)
                n += 1
    assert n > 500 and n_in > 50, (n, n_in)


def test_di_polyline_vertices_on_linear_solve_cubic(orc):
    """R7 step 6 (replaces round 1's dead check): the oracle's trajectory
    (di_traj + di_pos + di_vel) equals the cubic of an independent 4x4 linear
    solve at every polyline vertex t_k = k tau / Kc and every heuristic step
    t_k = k Delta, and reaches (p1, v1) at tau."""
    p = _tiny("c3", 150)
    rm = orc.build_roadmap(p)
    d = 3
    checked = 0
    for u in range(0, p.n, 5):
        for e in range(rm["row_ptr"][u], rm["row_ptr"][u + 1]):
            v = int(rm["dst"][e])
            tau = float(rm["tau"][e])
            su, sv = p.samples[u], p.samples[v]
            A = _cubic_np(su, sv, d, tau)
            Kc = max(1, math.ceil(tau / p.params["collision_dt"]))
            K = max(1, math.ceil(tau / p.params["dt"]))
            ts = np.concatenate([(np.arange(Kc + 1) * tau) / Kc, np.arange(K) * (tau / K)])
            scale = 1.0 + np.abs(su[:2 * d]).max() + np.abs(sv[:2 * d]).max()
            for t in ts[:: max(1, len(ts) // 12)]:
                x, vel = orc.di_state(su, sv, d, tau, t)
                assert np.abs(x - _pos(A, [t])[0]).max() <= 1e-12 * scale * (1 + tau) ** 3
                assert np.abs(vel - _vel(A, [t])[0]).max() <= 1e-12 * scale * (1 + tau) ** 3
            x, vel = orc.di_state(su, sv, d, tau, tau)
            assert np.abs(x - sv[:d]).max() <= 1e-12 * scale * (1 + tau) ** 3
            assert np.abs(vel - sv[d:2 * d]).max() <= 1e-12 * scale * (1 + tau) ** 3
            checked += 1
    assert checked > 50


# ---------------------------------------------------------------------------
# (c) FOV cone around the interpolated heading, R9 / P:319
# ---------------------------------------------------------------------------

def _heading_problem(features, h0, h1):
    east = (math.cos(h0), math.sin(h0))
    end = (math.cos(h1), math.sin(h1))
    return line_problem([(0.0, 0.0, 1.5, 0.0, 0.0, 0.0, *east), (2.0, 0.0, 1.5, 0.0, 0.0, 0.0, *end)],
                        features=features, heuristic=2, max_range=100.0)


def _expected_counts(prob, tau, K):
    """Visible features per step from angles: heading direction atan2 of the
    nlerp (1 - s) h_u + s h_v, bearing atan2 of the feature from the cubic's
    position; visible iff the horizontal angle difference is <= 45 deg
    (features at the vehicle's height, no obstacles).  Returns counts and a
    mask of steps with every feature > 1e-6 rad from the cone's edge."""
    su, sv = prob.samples[0], prob.samples[1]
    A = _cubic_np(su, sv, 3, tau)
    Dl = tau / K
    cnt = np.zeros(K, int)
    ok = np.ones(K, bool)
    for k in range(K):
        t = k * Dl
        s = t / tau
        hx = (1 - s) * su[6] + s * sv[6]
        hy = (1 - s) * su[7] + s * sv[7]
        th = math.atan2(hy, hx)
        x = _pos(A, [t])[0]
        for f in prob.features:
            ph = math.atan2(f[1] - x[1], f[0] - x[0])
            dang = abs((ph - th + math.pi) % (2 * math.pi) - math.pi)
            if abs(dang - math.pi / 4) < 1e-6:
                ok[k] = False
            cnt[k] += dang <= math.pi / 4
    return cnt, ok


@pytest.mark.parametrize("h0,h1,feats", [
    (0.0, math.pi / 2, [[1.0, 3.0, 1.5]]),                  # visible only under the end heading
    (math.pi / 2, 0.0, [[1.0, 3.0, 1.5]]),                  # visible only under the start heading
    (0.0, math.pi / 2, [[1.0, 3.0, 1.5], [6.0, 0.0, 1.5]]),  # one feature gained, one lost
    (-2.5, 2.0, [[-3.0, -2.0, 1.5], [0.5, 4.0, 1.5], [-2.0, 3.0, 1.5]]),
])
def test_heading_fov_follows_interpolated_yaw(orc, h0, h1, feats):
    """Distinct start and end headings: the oracle's per-step visible counts
    (recovered from the count increments, Delta - k Delta / n_f) equal the
    angle-based counts on the interpolated heading, and both values occur, so
    a reversed interpolation (s <-> 1 - s) or a constant heading fails."""
    prob = _heading_problem(feats, h0, h1)
    ed = orc.edge(prob, 0, 1)
    assert ed is not None and ed["coll"] == 0
    inc = orc.edge_increments(prob, 0, 1, ed["c64"], ed["tau"])
    K = len(inc)
    Dl = ed["tau"] / K
    nf = prob.params["n_f"]
    got = np.rint((Dl - inc) * nf / Dl).astype(int)
    want, ok = _expected_counts(prob, ed["tau"], K)
    assert ok.sum() >= K - 2
    assert np.array_equal(got[ok], want[ok]), (got, want)
    assert len(set(want.tolist())) >= 2
    # the reversed interpolation would give a different per-step pattern
    rev = _heading_problem(feats, h1, h0)
    want_rev, _ = _expected_counts(rev, ed["tau"], K)
    assert not np.array_equal(got, want_rev)


@pytest.mark.parametrize("p0,v0,p1,v1", [
    ((0.0, 0.0, 1.5), (0.5, 0.5, 0.0), (2.0, 0.5, 1.5), (0.5, -0.5, 0.0)),
    ((0.0, 0.0, 1.0), (0.0, 0.0, 0.3), (1.5, -1.0, 2.0), (-0.4, 0.2, 0.0)),
])
def test_di_collision_targeted_boxes(orc, p0, v0, p1, v1):
    """R8 vertex placement: a 2 mm box centred on the midpoint of each segment
    of the independent polyline (vertices p(k tau / Kc) of the linear-solve
    cubic), and one just before the final vertex, must collide; the same box
    moved 3 cm sideways must not.  A polyline through other vertex times (e.g.
    k tau / (Kc + 1)) or a wrong cubic coefficient misses the boxes."""
    east = (1.0, 0.0)
    base = line_problem([(*p0, *v0, *east), (*p1, *v1, *east)])
    ed = orc.edge(base, 0, 1)
    assert ed is not None and ed["coll"] == 0
    tau = ed["tau"]
    Kc = max(1, math.ceil(tau / base.params["collision_dt"]))
    assert Kc >= 5
    A = _cubic_np(base.samples[0], base.samples[1], 3, tau)
    V = _pos(A, np.arange(Kc + 1) * tau / Kc)
    pts = [(k, 0.5) for k in range(Kc)] + [(Kc - 1, 0.97)]
    for k, f in pts:
        P = V[k] + f * (V[k + 1] - V[k])
        d = V[k + 1] - V[k]
        side = np.array([-d[1], d[0], 0.0])
        side = side / np.linalg.norm(side) if np.linalg.norm(side) > 0 else np.array([0.0, 0.0, 1.0])
        for off, want in ((0.0, 1), (0.03, 0)):
            c = P + off * side
            prob = line_problem([(*p0, *v0, *east), (*p1, *v1, *east)],
                                obstacles=[[*(c - 1e-3), *(c + 1e-3)]])
            assert orc.collision(prob, 0, 1, tau) == bool(want), (k, f, off)
