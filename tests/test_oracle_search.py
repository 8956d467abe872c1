"""Pins of the oracle's Alg. 3 (Explore).

* exact regime (lambda r_n <= w_min / 2): the result is
  the plain definition -- the minimum-cost walk whose every node prefix has
  h <= beta -- so it must equal brute-force enumeration of walks and, at
  beta = inf, scipy's Dijkstra;
* literal-semantics worked examples where lambda = 0.5 departs from the
  optimum (early termination), the closed group boundary (A3.18),
  strict-cost dominance and the mid-wave goal rule (A3.5);
* invariants of returned plans on the C1/C2 roadmaps.
"""
import math

import numpy as np
import pytest
import scipy.sparse as sp
from scipy.sparse.csgraph import dijkstra

from synth import load_config, make_problem
from graphs import csr, random_graph  # noqa: F401

INF = float("inf")


def run(orc, g, goal_nodes, beta, lam, r, start=0):
    goal = np.zeros(g["n"], np.uint8)
    goal[list(goal_nodes)] = 1
    return orc.search_csr(g["n"], g["row_ptr"], g["dst"], g["coll"], g["w"], g["s"], g["c"], goal, start, beta,
                          lam, r)


# ---------------------------------------------------------------------------
# brute force (plain definition of Eq. 2 restricted to nodes, R11)
# ---------------------------------------------------------------------------

def brute_force(g, goal_nodes, beta, max_len):
    """Minimum over walks from node 0 of (cost, h, node sequence) among walks
    whose prefix h <= beta at every node; f32 arithmetic in path order, the
    edge map h -> max(c, h + s) (R10)."""
    best = None
    n = g["n"]
    adj = [[] for _ in range(n)]
    for u in range(n):
        for e in range(g["row_ptr"][u], g["row_ptr"][u + 1]):
            if not g["coll"][e]:
                adj[u].append((int(g["dst"][e]), g["w"][e], g["s"][e], g["c"][e]))
    stack = [(0, np.float32(0), np.float32(0), (0,))]
    while stack:
        u, cost, h, path = stack.pop()
        if best is not None and cost > best[0]:
            continue
        if u in goal_nodes:
            key = (cost, h, path)
            if best is None or key < best:
                best = key
        if len(path) > max_len:
            continue
        for (v, w, s, c) in adj[u]:
            nc = np.float32(cost + w)
            t = np.float32(h + s)
            nh = t if t > c else c
            if float(nh) <= beta:
                stack.append((v, nc, nh, path + (v,)))
    return best


@pytest.mark.parametrize("seed", range(20))
def test_exact_regime_equals_brute_force(orc, seed):
    """SPEC S:477 / north_star: on tiny graphs the exact-regime result equals
    brute-force enumeration (walks up to 2n edges, R27), finite beta."""
    rng = np.random.default_rng(100 + seed)
    n = int(rng.integers(4, 7))
    g = random_graph(rng, n, 3)
    goal_nodes = {n - 1}
    r = 1.0
    wmin = float(g["w"].min())
    lam = wmin / (2.0 * r)
    for beta in [INF, 1.0, 0.5, 0.25]:
        bf = brute_force(g, goal_nodes, beta, 2 * n)
        res = run(orc, g, goal_nodes, beta, lam, r)
        if bf is None:
            assert res["status_str"] == "NO_FEASIBLE_PLAN"
            continue
        assert res["status_str"] == "OK"
        assert res["cost"] == bf[0], (beta, res["cost"], bf)
        assert res["h"] == bf[1]
        assert tuple(res["path"].tolist()) == bf[2]


@pytest.mark.parametrize("seed", range(20))
def test_exact_regime_equals_dijkstra(orc, seed):
    """SPEC S:476 (corrected to the exact regime): beta = inf -> cost equals
    Dijkstra's on the same f32 weights (1e-6 relative: f32 vs f64 sums)."""
    rng = np.random.default_rng(seed)
    n = int(rng.integers(20, 200))
    g = random_graph(rng, n, int(rng.integers(2, 6)))
    free = g["coll"] == 0
    rows = np.repeat(np.arange(n), np.diff(g["row_ptr"]))
    M = sp.csr_matrix((g["w"][free].astype(np.float64), (rows[free], g["dst"][free])), shape=(n, n))
    dist = dijkstra(M, directed=True, indices=0)
    goal = int(rng.integers(1, n))
    lam = float(g["w"].min()) / 2.0
    res = run(orc, g, {goal}, INF, lam, 1.0)
    if math.isinf(dist[goal]):
        assert res["status_str"] == "NO_FEASIBLE_PLAN"
    else:
        assert res["status_str"] == "OK"
        assert abs(float(res["cost"]) - dist[goal]) <= 1e-6 * dist[goal]


# ---------------------------------------------------------------------------
# literal semantics at lambda = 0.5
# ---------------------------------------------------------------------------

def test_early_termination_example(orc):
    """P:230-231 ("potential for ... early termination"): s->g costs 0.99 r;
    the chain s->1->2->3->4->g costs 0.01 r per edge.  lambda = 0.5 returns
    the 0.99 plan; lambda = 0.01 returns the optimal 0.05 chain."""
    edges = [(0, 5, 0.99, 0, 0), (0, 1, 0.01, 0, 0), (1, 2, 0.01, 0, 0), (2, 3, 0.01, 0, 0),
             (3, 4, 0.01, 0, 0), (4, 5, 0.01, 0, 0)]
    g = csr(6, edges)
    a = run(orc, g, {5}, INF, 0.5, 1.0)
    assert a["path"].tolist() == [0, 5] and a["cost"] == np.float32(0.99)
    b = run(orc, g, {5}, INF, 0.01, 1.0)
    assert b["path"].tolist() == [0, 1, 2, 3, 4, 5]
    assert abs(float(b["cost"]) - 0.05) < 1e-6


def test_group_boundary_is_closed(orc):
    """A3.18 uses p.cost <= i lambda r_n: a plan of cost exactly T joins
    G_1.  Here that expands node 2 and returns 0.7 via [0,2,3]; SPEC's
    half-open bucket_index would return 0.9 via [0,3]."""
    g = csr(4, [(0, 2, 0.5, 0, 0), (0, 3, 0.9, 0, 0), (2, 3, 0.2, 0, 0)])
    res = run(orc, g, {3}, INF, 0.5, 1.0)
    assert res["path"].tolist() == [0, 2, 3]
    assert res["cost"] == np.float32(np.float32(0.5) + np.float32(0.2))


def test_equal_pairs_both_survive(orc):
    """P:193 dominance is strict in cost: equal (cost, h) plans both stay in P.
    Both reach node 3 in wave 2 (inserted == 2) and the lexicographic tie-break
    (R16) returns [0, 1, 3]."""
    g = csr(5, [(0, 1, 0.25, 0, 0), (0, 2, 0.25, 0, 0), (1, 3, 0.25, 0, 0), (2, 3, 0.25, 0, 0),
                (3, 4, 0.25, 0, 0)])
    res = run(orc, g, {4}, INF, 0.5, 1.0)
    wc = res["wave_counters"]
    assert res["path"].tolist() == [0, 1, 3, 4]
    # wave 2 (G_1 = {@1, @2}) inserts two labels at node 3
    assert wc[1][4] == 2
    # a strictly dominated twin is removed: make 2->3 cost more, same h
    g2 = csr(5, [(0, 1, 0.25, 0, 0), (0, 2, 0.25, 0, 0), (1, 3, 0.25, 0, 0), (2, 3, 0.3, 0, 0),
                 (3, 4, 0.25, 0, 0)])
    assert run(orc, g2, {4}, INF, 0.5, 1.0)["wave_counters"][1][4] == 1


def test_mid_wave_goal_does_not_stop_wave(orc):
    """A3.5 tests the group before expansion: a goal plan created mid-wave does
    not stop the wave (R13); every plan of G is expanded."""
    g = csr(4, [(0, 1, 0.1, 0, 0), (0, 2, 0.1, 0, 0), (1, 3, 0.1, 0, 0), (2, 0, 0.1, 0, 0), (2, 1, 0.1, 0, 0)])
    res = run(orc, g, {3}, INF, 0.5, 1.0)
    # wave 1: root -> 2 relaxations; wave 2: G_1 = {@1, @2} -> 1 + 2 relaxations
    assert res["wave_counters"][:, 2].tolist() == [2, 3]
    assert res["relaxations"] == 5


def test_start_in_goal_and_infeasible(orc):
    g = csr(2, [(0, 1, 0.5, 0.1, 0.1)])
    a = run(orc, g, {0}, INF, 0.5, 1.0)
    assert a["path"].tolist() == [0] and a["cost"] == 0 and a["waves"] == 0
    b = run(orc, g, {1}, 0.0, 0.5, 1.0)      # beta = 0, positive profile
    assert b["status_str"] == "NO_FEASIBLE_PLAN"
    c = run(orc, csr(2, [(0, 1, 0.5, 0.0, 0.0)]), {1}, 0.0, 0.5, 1.0)
    assert c["status_str"] == "OK" and c["h"] == 0.0


def test_two_corridor_homotopy_switch(orc):
    """S:296 / S:478 (Fig. 1 pattern): a short feature-poor corridor
    and a long feature-rich one; beta = inf takes the short one, a tight beta
    the long one at higher cost."""
    edges = [(0, 1, 0.3, 0.3, 0.3), (1, 2, 0.3, 0.3, 0.3), (2, 5, 0.3, 0.3, 0.3),
             (0, 3, 0.5, 0.05, 0.05), (3, 4, 0.5, -0.05, 0.0), (4, 5, 0.5, 0.05, 0.05)]
    g = csr(6, edges)
    a = run(orc, g, {5}, INF, 0.5, 1.0)
    b = run(orc, g, {5}, 0.2, 0.5, 1.0)
    assert a["path"].tolist() == [0, 1, 2, 5]
    assert b["path"].tolist() == [0, 3, 4, 5]
    assert float(b["cost"]) > float(a["cost"])


def test_weighted_sum_fails_where_multiobjective_succeeds(orc):
    """Fig. 2: through a single-file passage node 2, plan A (cheap,
    h = 0.6) beats plan B (costly, h = 0) under any weighted sum with w < 1,
    and A's continuation violates beta; Explore keeps both and succeeds."""
    edges = [(0, 1, 0.2, 0.6, 0.6), (1, 2, 0.2, 0.0, 0.0), (0, 3, 0.6, 0.0, 0.0), (3, 2, 0.6, 0.0, 0.0),
             (2, 4, 0.2, 0.5, 0.5)]
    g = csr(5, edges)
    res = run(orc, g, {4}, 0.9, 0.5, 1.0)
    assert res["path"].tolist() == [0, 3, 2, 4]
    # weighted sum (single label per node, keep argmin of cost + w h): picks A at node 2
    for wgt in [0.0, 0.5, 0.9]:
        a = 0.4 + wgt * 0.6
        b = 1.2 + wgt * 0.0
        assert a < b          # the scalarised search would keep only A, whose extension has h = 1.1 > beta


# ---------------------------------------------------------------------------
# invariants on the C1 / C2 roadmaps
# ---------------------------------------------------------------------------

@pytest.fixture(scope="module")
def c1(orc):
    p = make_problem(load_config("c1"))
    return p, orc.build_roadmap(p)


def check_plan_invariants(p, rm, res, beta):
    path = res["path"].tolist()
    assert path[0] == p.start
    cost = np.float32(0)
    h = np.float32(0)
    hp = np.float32(0)
    for a, b in zip(path[:-1], path[1:]):
        seg = range(rm["row_ptr"][a], rm["row_ptr"][a + 1])
        es = [e for e in seg if rm["dst"][e] == b]
        assert len(es) == 1
        e = es[0]
        assert rm["coll"][e] == 0
        cost = np.float32(cost + rm["w"][e])
        t = np.float32(h + rm["s"][e])
        h = t if t > rm["c"][e] else rm["c"][e]
        assert float(h) <= beta                      # prefix feasibility (A3.9)
        hp = max(hp, h)
    assert cost == res["cost"] and h == res["h"] and hp == res["h_peak"]
    pos = p.samples[path[-1], :p.pos_dim]
    assert np.all(pos >= p.goal_lo) and np.all(pos <= p.goal_hi)


@pytest.mark.parametrize("beta", [INF, 0.3, 0.22])
def test_c1_plan_invariants(orc, c1, beta):
    p, rm = c1
    res = orc.search(rm, p, beta)
    assert res["status_str"] == "OK"
    check_plan_invariants(p, rm, res, beta)
    wc = res["wave_counters"]
    assert wc[:, 2].sum() == res["relaxations"]
    assert wc[:, 4].sum() == res["labels_inserted"]
    assert np.all(wc[:, 3] <= wc[:, 2]) and np.all(wc[:, 4] <= wc[:, 3])


def test_c1_exact_regime_beta_monotone(orc, c1):
    """S:309 in the exact regime: tighter beta never lowers the returned cost."""
    p, rm = c1
    wmin = float(rm["w"][rm["coll"] == 0].min())
    lam = wmin / (2 * p.r)
    costs = []
    for beta in [INF, 0.3, 0.25, 0.22, 0.2]:
        res = orc.search(rm, p, beta, lam=lam)
        costs.append(float(res["cost"]) if res["status_str"] == "OK" else INF)
    assert all(a <= b for a, b in zip(costs, costs[1:]))
    # beta = inf in the exact regime equals Dijkstra on the roadmap
    n = p.n
    free = rm["coll"] == 0
    rows = np.repeat(np.arange(n), np.diff(rm["row_ptr"]))
    M = sp.csr_matrix((rm["w"][free].astype(np.float64), (rows[free], rm["dst"][free])), shape=(n, n))
    dist = dijkstra(M, directed=True, indices=0)
    goal = orc.goal_mask(p).astype(bool)
    assert abs(costs[0] - dist[goal].min()) <= 1e-6 * costs[0]


def test_e_rows_counter(orc, c1):
    """SURVEY §8(d) E_rows = per wave, the collision-free CSR entries of the
    DISTINCT head nodes of G_i.  Pins: a chain graph (one label per node, so
    E_rows = relaxations, wave by wave); on C1, E_rows <= relaxations per wave
    and a wave with #G_i = 1 has E_rows = relax, while waves whose heads carry
    several labels read each row once (E_rows < relaxations in total)."""
    g = csr(4, [(0, 1, 1.0, 0.0, 0.0), (1, 2, 1.0, 0.0, 0.0), (2, 3, 1.0, 0.0, 0.0), (1, 3, 5.0, 0.0, 0.0)])
    r = run(orc, g, [3], INF, 0.5, 1.0)
    assert r["e_rows_per_wave"] == r["wave_counters"][:, 2].tolist()
    p, rm = c1
    res = orc.search(rm, p, 0.3)
    wc = res["wave_counters"]
    er = np.asarray(res["e_rows_per_wave"])
    assert np.all(er <= wc[:, 2]) and er.sum() == res["e_rows"]
    assert np.all(er[wc[:, 1] == 1] == wc[wc[:, 1] == 1, 2])
    assert er.sum() < wc[:, 2].sum()      # some heads carry several labels at beta = 0.3
