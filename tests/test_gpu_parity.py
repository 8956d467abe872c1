"""GPU parity: libmpap.so (sm_100a kernels, through the C ABI) vs the CPU
oracle on identical seeded inputs.

Bar (BASELINE.json north_star): roadmap adjacency, collision
bits and the plan's node sequence bit-exact; cost and perception value
bit-exact (stronger than the 1e-5 relative the north star allows); per-wave
counters equal.  Small cases run the oracle in-test; full sizes compare with
tests/golden/*.json written by tests/golden/make_golden.py (oracle only) and
with rows the oracle computes one by one.
"""
import json
import os

import numpy as np
import pytest

from synth import load_config, make_problem

pytestmark = pytest.mark.gpu
INF = float("inf")
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


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


def bits(a):
    a = np.ascontiguousarray(a)
    return a.view(np.uint32) if a.dtype == np.float32 else a


def assert_roadmap_equal(g, o):
    assert np.array_equal(g["row_ptr"], o["row_ptr"]), "row_ptr"
    assert np.array_equal(g["dst"], o["dst"]), "dst"
    assert np.array_equal(g["coll"], o["coll"]), "coll"
    for k in ("w", "s", "c"):
        mism = np.nonzero(bits(g[k]) != bits(o[k]))[0]
        assert mism.size == 0, (k, mism[:10], g[k][mism[:5]], o[k][mism[:5]])


def assert_search_equal(g, o, counters=True):
    assert g["status"] == o["status"], (g["status_str"], o["status_str"])
    assert g["waves"] == o["waves"]
    assert g["relaxations"] == o["relaxations"]
    assert g["labels_inserted"] == o["labels_inserted"]
    if o["status"] == 0:
        assert g["path"].tolist() == o["path"].tolist()
        assert bits(np.float32(g["cost"])) == bits(np.float32(o["cost"]))
        assert bits(np.float32(g["h"])) == bits(np.float32(o["h"]))
        assert bits(np.float32(g["h_peak"])) == bits(np.float32(o["h_peak"]))
    if counters:
        assert np.array_equal(g["wave_counters"], o["wave_counters"]), (g["wave_counters"], o["wave_counters"])


def small(name, n=None, **over):
    cfg = load_config(name)
    if n is not None:
        cfg["n_samples"] = n
    cfg.update(over)
    return make_problem(cfg)


# ---------------------------------------------------------------------------
# roadmap build (Alg. 2 + heuristic): bit-exact CSR
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("name,n", [("c1", None), ("c1", 37), ("c2", None), ("c2", 90), ("c3", 500),
                                    ("c4", 300), ("c3", 2)])
def test_roadmap_parity(mp, orc, name, n):
    prob = small(name, n)
    rm = mp.pb.build_problem(prob)
    g = mp.mpap_roadmap_export(rm)
    o = orc.build_roadmap(prob)
    assert_roadmap_equal(g, o)
    info = mp.mpap_roadmap_info(rm)
    assert info["nnz"] == len(o["dst"]) and info["nnz_free"] == int((o["coll"] == 0).sum())


def test_roadmap_parity_heuristic_variants(mp, orc):
    """Every heuristic mode: omni / velocity-FOV on C2-like, heading count and
    MLP on C3-like inputs, kinematic + heading."""
    for name, heur in [("c2", 0), ("c2", 1), ("c3", 2), ("c3", 3), ("c3", 0)]:
        prob = small(name, 150)
        prob.heuristic = heur
        rm = mp.pb.build_problem(prob)
        assert_roadmap_equal(mp.mpap_roadmap_export(rm), orc.build_roadmap(prob))
    prob = small("c3", 150)
    prob.dynamics = 0
    prob.samples = np.ascontiguousarray(prob.samples[:, [0, 1, 2, 6, 7]])
    prob.r = 1.5
    rm = mp.pb.build_problem(prob)
    assert_roadmap_equal(mp.mpap_roadmap_export(rm), orc.build_roadmap(prob))


def test_roadmap_no_obstacles_no_features(mp, orc):
    prob = small("c2", 60)
    prob.obstacles = np.zeros((0, 4))
    prob.features = np.zeros((0, 2))
    rm = mp.pb.build_problem(prob)
    assert_roadmap_equal(mp.mpap_roadmap_export(rm), orc.build_roadmap(prob))


def test_full_size_rows_sampled(mp, orc):
    """C3 at BASELINE size (n = 4001): 24 sampled rows equal the oracle's
    row-by-row computation."""
    prob = make_problem(load_config("c3"))
    rm = mp.pb.build_problem(prob)
    g = mp.mpap_roadmap_export(rm)
    rng = np.random.default_rng(0)
    for u in rng.choice(prob.n, 24, replace=False):
        o = orc.build_row(prob, int(u))
        a, b = g["row_ptr"][u], g["row_ptr"][u + 1]
        assert np.array_equal(g["dst"][a:b], o["dst"])
        assert np.array_equal(g["coll"][a:b], o["coll"])
        for k in ("w", "s", "c"):
            assert np.array_equal(bits(g[k][a:b]), bits(o[k]))
    gold = json.load(open(os.path.join(GOLDEN, "c3_full.json")))
    info = mp.mpap_roadmap_info(rm)
    assert info["nnz"] == gold["nnz"] and info["nnz_free"] == gold["nnz_free"]


# ---------------------------------------------------------------------------
# search (Alg. 3)
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("name", ["c1", "c2"])
def test_search_parity_configs(mp, orc, name):
    prob = make_problem(load_config(name))
    rm = mp.pb.build_problem(prob)
    orm = orc.build_roadmap(prob)
    for beta in prob.betas:
        g = mp.pb.search_problem(rm, prob, beta, trace_waves=4096)
        o = orc.search(orm, prob, beta)
        assert_search_equal(g, o)


def test_search_parity_c3_reduced(mp, orc):
    prob = small("c3", 700)
    rm = mp.pb.build_problem(prob)
    orm = orc.build_roadmap(prob)
    for beta in [INF, 6.0, 3.0, 1.0]:
        assert_search_equal(mp.pb.search_problem(rm, prob, beta, trace_waves=4096), orc.search(orm, prob, beta))


def test_search_parity_lambda(mp, orc):
    """lambda in (0,1]: the exact regime and lambda = 1."""
    prob = make_problem(load_config("c1"))
    rm = mp.pb.build_problem(prob)
    orm = orc.build_roadmap(prob)
    wmin = float(orm["w"][orm["coll"] == 0].min())
    for lam in [wmin / (2 * prob.r), 0.25, 1.0]:
        for beta in [INF, 0.2174]:
            g = mp.pb.search_problem(rm, prob, beta, lam=lam, trace_waves=8192)
            o = orc.search(orm, prob, beta, lam=lam)
            assert_search_equal(g, o)


def _golden_check(mp, rm, prob, gold, env=0):
    for s in gold["searches"]:
        beta = INF if s["beta"] == "inf" else float(s["beta"])
        g = mp.pb.search_problem(rm, prob, beta, env=env, trace_waves=4096)
        assert g["status"] == s["status"]
        assert g["waves"] == s["waves"] and g["relaxations"] == s["relaxations"]
        assert g["labels_inserted"] == s["labels_inserted"]
        assert g["wave_counters"].tolist() == s["wave_counters"]
        if s["status"] == 0:
            assert g["path"].tolist() == s["path"]
            assert np.float32(g["cost"]).tobytes().hex() == s["cost"]
            assert np.float32(g["h"]).tobytes().hex() == s["h"]
            assert np.float32(g["h_peak"]).tobytes().hex() == s["h_peak"]


@pytest.mark.parametrize("l2_persist", [False, True])
def test_search_full_size_c3_golden(mp, monkeypatch, l2_persist):
    """C3 full size against the oracle's stored run; with l2_persist the
    search runs under the optional L2 access-policy window over the CSR
    (MPAP_SEARCH_L2_PERSIST), which must not change anything."""
    if l2_persist:
        monkeypatch.setenv("MPAP_SEARCH_L2_PERSIST", "1")
    prob = make_problem(load_config("c3"))
    rm = mp.pb.build_problem(prob)
    _golden_check(mp, rm, prob, json.load(open(os.path.join(GOLDEN, "c3_full.json"))))


def test_batch_full_size_c5_golden(mp):
    """One batched build of 8 C5 environments + one batched search of 8
    queries, vs the stored oracle results.  A batch of at most 8 queries runs
    query by query on the whole grid (search_batch_device); the bench's own
    64-query cluster launch and the 256-query one-CTA-per-query launch are
    compared in tests/test_gpu_fullsize.py."""
    cfg = load_config("c5")
    gold = json.load(open(os.path.join(GOLDEN, "c5_full.json")))["envs"]
    probs = [make_problem(cfg, env_index=k) for k in range(len(gold))]
    B = mp.pb.Batch(probs)
    rm = B.build()
    for e, gd in enumerate(gold):
        info = mp.mpap_roadmap_info(rm, e)
        assert info["nnz"] == gd["nnz"] and info["nnz_free"] == gd["nnz_free"]
    betas_list = [s["beta"] for s in gold[0]["searches"]]
    for bi, b in enumerate(betas_list):
        beta = INF if b == "inf" else float(b)
        paths, res = B.search(rm, [beta] * len(probs), path_capacity=512)
        for e, gd in enumerate(gold):
            s = gd["searches"][bi]
            assert res[e]["status"] == s["status"], (e, res[e])
            assert res[e]["waves"] == s["waves"] and res[e]["relaxations"] == s["relaxations"]
            assert res[e]["labels_inserted"] == s["labels_inserted"]
            if s["status"] == 0:
                assert paths[e, : res[e]["path_len"]].tolist() == s["path"]
                assert np.float32(res[e]["cost"]).tobytes().hex() == s["cost"]
                assert np.float32(res[e]["h"]).tobytes().hex() == s["h"]
    # per-environment single searches through the batch roadmap agree too
    _golden_check(mp, rm, probs[1], gold[1], env=1)


def test_batch_ragged_equals_single(mp, orc):
    """Batch of environments with different n (ragged), mixed betas; every
    query equals the single-query result and the oracle."""
    cfg = load_config("c5")
    cfg["n_samples"] = 300
    probs = []
    for k, n in enumerate([300, 180, 1, 240]):
        c = dict(cfg)
        c["n_samples"] = n
        probs.append(make_problem(c, env_index=k))
    B = mp.pb.Batch(probs)
    rm = B.build()
    betas = [INF, 4.0, INF, 2.5]
    paths, res = B.search(rm, betas, path_capacity=256)
    for e, prob in enumerate(probs):
        orm = orc.build_roadmap(prob)
        assert_roadmap_equal(mp.mpap_roadmap_export(rm, e), orm)
        o = orc.search(orm, prob, betas[e])
        assert res[e]["status"] == o["status"]
        if o["status"] == 0:
            assert paths[e, : res[e]["path_len"]].tolist() == o["path"].tolist()
            assert np.float32(res[e]["cost"]) == o["cost"] and np.float32(res[e]["h"]) == o["h"]
        assert res[e]["relaxations"] == o["relaxations"]


# ---------------------------------------------------------------------------
# literal-semantics graphs through mpap_roadmap_import (same graphs as the
# oracle pins in tests/test_oracle_search.py)
# ---------------------------------------------------------------------------

def _import_and_compare(mp, orc, n, edges, goal_nodes, betas, lams, r=1.0):
    from graphs import csr
    g = csr(n, edges)
    pos = np.zeros((n, 2))
    pos[:, 0] = np.arange(n)
    goal = np.zeros(n, np.uint8)
    goal[list(goal_nodes)] = 1
    dc = g["dst"].astype(np.uint32) | (g["coll"].astype(np.uint32) << 31)
    rm = mp.mpap_roadmap_import(pos, g["row_ptr"], dc, g["w"], g["s"], g["c"], r)
    lo = [min(goal_nodes) - 0.25, -0.5]
    hi = [max(goal_nodes) + 0.25, 0.5]
    assert all(goal[x] == (lo[0] <= x <= hi[0]) for x in range(n)), "goal box must select exactly goal_nodes"
    for lam in lams:
        for beta in betas:
            gr = mp.mpap_search(rm, 0, 0, lo, hi, beta, lam, trace_waves=4096)
            o = orc.search_csr(n, g["row_ptr"], g["dst"], g["coll"], g["w"], g["s"], g["c"], goal, 0, beta, lam, r)
            assert_search_equal(gr, o)


def test_literal_graphs(mp, orc):
    _import_and_compare(mp, orc, 6, [(0, 5, 0.99, 0, 0), (0, 1, 0.01, 0, 0), (1, 2, 0.01, 0, 0), (2, 3, 0.01, 0, 0),
                                     (3, 4, 0.01, 0, 0), (4, 5, 0.01, 0, 0)], {5}, [INF], [0.5, 0.01])
    _import_and_compare(mp, orc, 4, [(0, 2, 0.5, 0, 0), (0, 3, 0.9, 0, 0), (2, 3, 0.2, 0, 0)], {3}, [INF], [0.5])
    _import_and_compare(mp, orc, 5, [(0, 1, 0.25, 0, 0), (0, 2, 0.25, 0, 0), (1, 3, 0.25, 0, 0), (2, 3, 0.25, 0, 0),
                                     (3, 4, 0.25, 0, 0)], {4}, [INF], [0.5])
    _import_and_compare(mp, orc, 4, [(0, 1, 0.1, 0, 0), (0, 2, 0.1, 0, 0), (1, 3, 0.1, 0, 0), (2, 0, 0.1, 0, 0),
                                     (2, 1, 0.1, 0, 0)], {3}, [INF], [0.5])
    _import_and_compare(mp, orc, 2, [(0, 1, 0.5, 0.1, 0.1)], {0}, [INF], [0.5])       # start in goal
    _import_and_compare(mp, orc, 2, [(0, 1, 0.5, 0.1, 0.1)], {1}, [0.0, INF], [0.5])  # beta = 0 infeasible
    _import_and_compare(mp, orc, 3, [(0, 1, 0.5, 0.0, 0.0, 1), (1, 2, 0.5, 0.0, 0.0)], {2}, [INF], [0.5])  # coll


@pytest.mark.parametrize("seed", range(12))
def test_random_graphs(mp, orc, seed):
    from graphs import random_graph
    rng = np.random.default_rng(500 + seed)
    n = int(rng.integers(5, 60))
    g = random_graph(rng, n, int(rng.integers(2, 7)), neg_frac=0.5)
    edges = [(u, int(g["dst"][e]), float(g["w"][e]), float(g["s"][e]), float(g["c"][e]), int(g["coll"][e]))
             for u in range(n) for e in range(g["row_ptr"][u], g["row_ptr"][u + 1])]
    goal = {n - 1}
    _import_and_compare(mp, orc, n, edges, goal, [INF, 1.0, 0.5, 0.2], [0.5, 0.1, 1.0])


def test_path_buffer_too_small(mp):
    from graphs import csr
    g = csr(4, [(0, 1, 0.3, 0, 0), (1, 2, 0.3, 0, 0), (2, 3, 0.3, 0, 0)])
    pos = np.zeros((4, 2))
    pos[:, 0] = np.arange(4)
    rm = mp.mpap_roadmap_import(pos, g["row_ptr"], g["dst"].astype(np.uint32), g["w"], g["s"], g["c"], 1.0)
    with pytest.raises(mp.MpapError) as ei:
        mp.mpap_search(rm, 0, 0, [2.9, -1], [3.1, 1], INF, 0.5, path_capacity=2)
    assert ei.value.status == mp.MPAP_ERR_BUFFER_TOO_SMALL


def test_no_goal_node(mp):
    prob = small("c1", 50)
    rm = mp.pb.build_problem(prob)
    with pytest.raises(mp.MpapError) as ei:
        mp.mpap_search(rm, 0, 0, [5.0, 5.0], [6.0, 6.0], INF, 0.5)
    assert ei.value.status == mp.MPAP_ERR_NO_GOAL_NODE


def test_device_resident_inputs_equal_host(mp):
    """mem = DEVICE (torch tensors) gives the same roadmap and plans as HOST."""
    import torch
    cfg = load_config("c5")
    cfg["n_samples"] = 400
    probs = [make_problem(cfg, env_index=k) for k in range(3)]
    B = mp.pb.Batch(probs)
    rm_h = B.build()
    dev = torch.device("cuda")
    rm_d = B.build(torch.from_numpy(B.samples).to(dev), torch.from_numpy(B.obstacles).to(dev),
                   torch.from_numpy(B.features).to(dev))
    for e in range(3):
        a, b = mp.mpap_roadmap_export(rm_h, e), mp.mpap_roadmap_export(rm_d, e)
        assert_roadmap_equal(a, b)
    paths_d = torch.zeros((3, 128), dtype=torch.int32, device=dev)
    res_d = torch.zeros(3 * 48, dtype=torch.uint8, device=dev)
    B.search(rm_d, [INF] * 3, path_capacity=128, paths=paths_d, results=res_d)
    torch.cuda.synchronize()
    ph, rh = B.search(rm_h, [INF] * 3, path_capacity=128)
    rd = res_d.cpu().numpy().view(mp.RESULT_DTYPE)
    pd = paths_d.cpu().numpy()
    assert np.array_equal(rd, rh)
    for e in range(3):   # rows beyond path_len are unspecified (include/mpap.h)
        n = rh[e]["path_len"]
        assert np.array_equal(pd[e, :n], ph[e, :n])


# ---------------------------------------------------------------------------
# NEXT-2: batched beta sweep / refinement on one roadmap
# ---------------------------------------------------------------------------

def test_beta_sweep_equals_single_and_oracle(mp, orc):
    prob = make_problem(load_config("c2"))
    rm = mp.pb.build_problem(prob)
    orm = orc.build_roadmap(prob)
    betas = [INF, 2.0, 1.5, 1.1762, 1.0, 0.9598, 0.93, 0.9, 0.5, 0.0]
    paths, res = mp.pb.beta_sweep(rm, prob, betas)
    for k, beta in enumerate(betas):
        o = orc.search(orm, prob, beta)
        assert res[k]["status"] == o["status"]
        assert res[k]["relaxations"] == o["relaxations"] and res[k]["waves"] == o["waves"]
        if o["status"] == 0:
            assert paths[k, : res[k]["path_len"]].tolist() == o["path"].tolist()
            assert np.float32(res[k]["cost"]) == o["cost"] and np.float32(res[k]["h"]) == o["h"]


def test_refine_beta_min_brackets_oracle_feasibility(mp, orc):
    """The refined bracket agrees with the oracle: infeasible at lo, feasible
    at hi (Explore feasibility is decided identically on both sides)."""
    prob = make_problem(load_config("c1"))
    rm = mp.pb.build_problem(prob)
    orm = orc.build_roadmap(prob)
    lo, hi, rounds = mp.pb.refine_beta_min(rm, prob, hi=1.0, rel_tol=1e-4)
    assert hi - lo <= 1e-4 * hi and rounds <= 6
    assert orc.search(orm, prob, hi)["status"] == 0
    assert orc.search(orm, prob, lo)["status"] == 3


def test_search_full_size_c4_golden(mp):
    """C4 (n = 16001, 200 boxes, 400 features) at BASELINE size: the whole-grid
    single-query search vs the stored oracle results (beta = inf and
    2 x beta_min)."""
    prob = make_problem(load_config("c4"))
    rm = mp.pb.build_problem(prob)
    gold = json.load(open(os.path.join(GOLDEN, "c4_full.json")))
    info = mp.mpap_roadmap_info(rm)
    assert info["nnz"] == gold["nnz"] and info["nnz_free"] == gold["nnz_free"]
    _golden_check(mp, rm, prob, gold)


def test_many_goal_ties(mp, orc):
    """More (cost, h) ties at the goal than the 32-entry tie list (R16): 48
    goal nodes reached at identical cost and h through 2-hop chains; the
    lexicographically smallest node sequence must win, as in the oracle
    (which scans every tie).  Ties are reached via intermediate nodes with
    descending ids so the winner is not the first goal node."""
    n_goal = 48
    n = 1 + 2 * n_goal
    edges = []
    for k in range(n_goal):
        mid = n_goal - k          # intermediate nodes 1..48 (descending)
        goalk = n_goal + 1 + k    # goal nodes 49..96
        edges.append((0, mid, 0.25, 0.0, 0.0))
        edges.append((mid, goalk, 0.25, 0.0, 0.0))
    goal = set(range(n_goal + 1, n))
    _import_and_compare(mp, orc, n, edges, goal, [INF, 1.0], [0.5, 1.0])
