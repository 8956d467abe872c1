"""NEXT-3 pins: the "for all t" perception constraint of Eq. 2 along
an edge, via the peak summary (S, C) (reading R10)."""
import numpy as np
import pytest

from graphs import csr

INF = float("inf")


def test_peak_summary_equals_stepwise_peak(orc):
    """max(C, h0 + S) is the largest value the stepwise clamp fold reaches from
    h0 (prefix 0 included): bit-exact for dyadic increments, 1e-12 otherwise."""
    rng = np.random.default_rng(21)
    for _ in range(300):
        K = int(rng.integers(1, 60))
        inc = rng.integers(-64, 65, K) / 1024.0
        S, C = orc.fold_peak(inc)
        s, c = orc.fold_summary(inc)
        assert S >= max(s, 0.0) and C >= c
        for h0 in [0.0, 0.015625, 0.25, float(rng.integers(0, 200)) / 256.0]:
            assert max(C, h0 + S) == orc.fold_stepwise_peak(h0, inc)
            assert max(C, h0 + S) >= orc.fold_stepwise(h0, inc)
        inc2 = rng.uniform(-0.05, 0.05, K)
        S2, C2 = orc.fold_peak(inc2)
        for h0 in [0.0, 0.01, 0.3]:
            assert abs(max(C2, h0 + S2) - orc.fold_stepwise_peak(h0, inc2)) < 1e-12


def _peak_graph(edges):
    """edges: (u, v, w, inc list) -> csr with s, c, S, C from the oracle's folds."""
    rows = []
    S, Cp = {}, {}
    for (u, v, w, inc) in edges:
        s, c = _orc.fold_summary(inc)
        Sp, Cq = _orc.fold_peak(inc)
        rows.append((u, v, w, s, c))
        S[(u, v)] = Sp
        Cp[(u, v)] = Cq
    n = 1 + max(max(e[0], e[1]) for e in edges)
    g = csr(n, rows)
    g["S"] = np.array([S[(u, int(g["dst"][e]))] for u in range(n) for e in range(g["row_ptr"][u], g["row_ptr"][u + 1])],
                      np.float32)
    g["C"] = np.array([Cp[(u, int(g["dst"][e]))] for u in range(n) for e in range(g["row_ptr"][u], g["row_ptr"][u + 1])],
                      np.float32)
    return g


_orc = None


@pytest.fixture(autouse=True)
def _bind(orc):
    global _orc
    _orc = orc


def _run(orc, g, goal, beta, forall_t, lam=0.5):
    gm = np.zeros(g["n"], np.uint8)
    gm[list(goal)] = 1
    return orc.search_csr(g["n"], g["row_ptr"], g["dst"], g["coll"], g["w"], g["s"], g["c"], gm, 0, beta, lam, 1.0,
                          S=g["S"], Cp=g["C"], forall_t=forall_t)


def test_forall_rejects_an_intra_edge_peak(orc):
    """An edge whose fold rises to 0.5 and returns to 0 satisfies the node-only
    bound 0.3 (R11) but not Eq. 2's bound for all t; the detour does."""
    g = _peak_graph([(0, 2, 0.3, [0.25, 0.25, -0.25, -0.25]),      # peak 0.5, final 0
                     (0, 1, 0.3, [0.125, 0.0]), (1, 2, 0.3, [0.0, -0.125])])
    a = _run(orc, g, {2}, 0.3, False)
    b = _run(orc, g, {2}, 0.3, True)
    assert a["path"].tolist() == [0, 2]
    assert b["path"].tolist() == [0, 1, 2]
    c = _run(orc, g, {2}, 0.1, True)
    assert c["status_str"] == "NO_FEASIBLE_PLAN"


def _brute(g, goal, beta, max_len):
    n = g["n"]
    adj = [[] for _ in range(n)]
    for u in range(n):
        for e in range(g["row_ptr"][u], g["row_ptr"][u + 1]):
            if not g["coll"][e]:
                adj[u].append((int(g["dst"][e]), g["w"][e], g["s"][e], g["c"][e], g["S"][e], g["C"][e]))
    best = None
    stack = [(0, np.float32(0), np.float32(0), (0,))]
    while stack:
        u, cost, h, path = stack.pop()
        if best is not None and cost > best[0]:
            continue
        if u in goal:
            key = (cost, h, path)
            if best is None or key < best:
                best = key
        if len(path) > max_len:
            continue
        for (v, w, s, c, S, C) in adj[u]:
            t = np.float32(h + s)
            nh = t if t > c else c
            t2 = np.float32(h + S)
            pk = t2 if t2 > C else C
            if float(nh) <= beta and float(pk) <= beta:
                stack.append((v, np.float32(cost + w), nh, path + (v,)))
    return best


@pytest.mark.parametrize("seed", range(12))
def test_forall_exact_regime_equals_brute_force(orc, seed):
    rng = np.random.default_rng(900 + seed)
    n = int(rng.integers(4, 7))
    edges = []
    for u in range(n):
        for v in rng.choice([x for x in range(n) if x != u], size=3, replace=False):
            K = int(rng.integers(1, 6))
            inc = (rng.integers(-16, 24, K) / 64.0).tolist()
            edges.append((u, int(v), float(rng.uniform(0.1, 1.0)), inc))
    g = _peak_graph(edges)
    lam = float(g["w"].min()) / 2.0
    for beta in [INF, 1.0, 0.6, 0.4]:
        bf = _brute(g, {n - 1}, beta, 2 * n)
        res = _run(orc, g, {n - 1}, beta, True, lam=lam)
        if bf is None:
            assert res["status_str"] == "NO_FEASIBLE_PLAN"
        else:
            assert res["status_str"] == "OK"
            assert res["cost"] == bf[0] and res["h"] == bf[1]
            assert tuple(res["path"].tolist()) == bf[2]


def test_forall_never_cheaper_on_c1(orc):
    """The all-t constraint only removes plans: in the exact regime its cost is
    never below the node-only cost, and equal at beta = inf."""
    from synth import load_config, make_problem
    p = make_problem(load_config("c1"))
    rm = orc.build_roadmap(p)
    wmin = float(rm["w"][rm["coll"] == 0].min())
    lam = wmin / (2 * p.r)
    for beta in [INF, 0.3, 0.25]:
        a = orc.search(rm, p, beta, lam=lam)
        b = orc.search(rm, p, beta, lam=lam, forall_t=True)
        if b["status"] == 0:
            assert a["status"] == 0 and float(b["cost"]) >= float(a["cost"])
        if beta == INF:
            assert b["cost"] == a["cost"] and b["path"].tolist() == a["path"].tolist()
