"""Full-size parity of the launch configurations the product times
(VERDICT r01 "Missing 3"): the bench's rank-0 shard of 64 C5 environments
(BASELINE.json configs[4]) built as one batch, searched as the bench does (64
queries: one thread-block cluster per query) and as a 256-query batch (one
CTA per query), plus CSR digests of the full C3, C4 and C5 roadmaps -- all
against tests/golden/*.json written by tests/golden/make_golden.py, which
calls only the oracle (Alg. 2 + heuristic, Alg. 3 literal; PAPER.md
P:206-220).

Bit-exact bar: every CSR array (row_ptr, dst | coll << 31, w, s, c) by
SHA-256 digest; per query status, waves, relaxations, inserted labels, plan
node sequence, cost / h / h_peak bits, and the per-wave counters.  Which team
kind ran is asserted with mpap_search_launches."""
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


def _digests(mp, rm, env):
    import sys
    sys.path.insert(0, GOLDEN)
    from digest import csr_digests
    return csr_digests(mp.mpap_roadmap_export(rm, env))


def _hex(x):
    return np.float32(x).tobytes().hex()


def _check(res, paths, q, s, counters=None):
    assert res[q]["status"] == s["status"], (q, res[q])
    assert res[q]["waves"] == s["waves"] and res[q]["relaxations"] == s["relaxations"], (q, res[q])
    assert res[q]["labels_inserted"] == s["labels_inserted"], q
    if s["status"] == 0:
        assert paths[q, : res[q]["path_len"]].tolist() == s["path"], q
        assert _hex(res[q]["cost"]) == s["cost"] and _hex(res[q]["h"]) == s["h"], q
        assert _hex(res[q]["h_peak"]) == s["h_peak"], q
    if counters is not None:
        assert counters[q].tolist() == s["wave_counters"], q


@pytest.fixture(scope="module")
def bench_shard(mp):
    """The bench's rank-0 batch: C5 environments 0..63 in one batched build."""
    gold = json.load(open(os.path.join(GOLDEN, "c5_bench.json")))
    cfg = load_config("c5")
    probs = [make_problem(cfg, env_index=k) for k in range(len(gold["envs"]))]
    B = mp.pb.Batch(probs)
    rm = B.build()
    yield B, rm, gold
    rm.free()


def test_bench_shard_csr_digests(mp, bench_shard):
    B, rm, gold = bench_shard
    assert len(gold["envs"]) == int(load_config("c5")["queries_per_gpu"])
    for e, gd in enumerate(gold["envs"]):
        info = mp.mpap_roadmap_info(rm, e)
        assert info["nnz"] == gd["nnz"] and info["nnz_free"] == gd["nnz_free"], e
        assert _digests(mp, rm, e) == gd["digests"], e


def _betas(gold):
    return [INF if b == "inf" else float(b) for b in gold["betas"]]


def test_bench_shard_64_queries_cluster_teams(mp, bench_shard):
    """The bench's timed search: 64 queries at the bench bound, one
    thread-block cluster per query."""
    B, rm, gold = bench_shard
    beta = _betas(gold)[0]
    assert beta == float(load_config("c5")["betas"][1])
    before = mp.mpap_search_launches()
    paths, res = B.search(rm, [beta] * len(B.probs), path_capacity=512)
    after = mp.mpap_search_launches()
    assert after["cluster"] > before["cluster"] and after["cta"] == before["cta"] and after["grid"] == before["grid"]
    for q, gd in enumerate(gold["envs"]):
        _check(res, paths, q, gd["searches"][0])
    assert 0.3 < float((res["status"] == 0).mean()) < 0.9   # both outcomes are exercised


def test_bench_shard_64_queries_cluster_wave_counters(mp, bench_shard):
    """Per-wave counters of the same batch in the same (cluster) launch
    configuration, through mpap_search_batch_trace."""
    B, rm, gold = bench_shard
    beta = _betas(gold)[0]
    before = mp.mpap_search_launches()
    paths, res, wc = B.search(rm, [beta] * len(B.probs), path_capacity=512, trace_waves=256)
    assert mp.mpap_search_launches()["cluster"] > before["cluster"]
    for q, gd in enumerate(gold["envs"]):
        _check(res, paths, q, gd["searches"][0], counters=wc)


@pytest.mark.parametrize("trace", [False, True])
def test_bench_shard_256_queries_cta_teams(mp, bench_shard, trace):
    """64 environments x 4 bounds = 256 queries: more than the SMs can hold as
    clusters, so one CTA per query (k_search) runs."""
    B, rm, gold = bench_shard
    betas = _betas(gold)
    ne = len(B.probs)
    envs = np.repeat(np.arange(ne, dtype=np.int32), len(betas))
    bq = np.tile(np.asarray(betas), ne)
    before = mp.mpap_search_launches()
    out = B.search(rm, bq, path_capacity=512, envs=envs, trace_waves=256 if trace else 0)
    after = mp.mpap_search_launches()
    assert after["cta"] > before["cta"]   # (a regrow-and-retry round of few queries may use clusters)
    paths, res = out[0], out[1]
    wc = out[2] if trace else None
    for q in range(len(envs)):
        _check(res, paths, q, gold["envs"][envs[q]]["searches"][q % len(betas)], counters=wc)


def test_bench_shard_forced_cta_and_cluster(mp, bench_shard, monkeypatch):
    """The other team kinds on the same queries: 64 queries forced to one CTA
    each (MPAP_SEARCH_CTA), and 8 queries forced off the whole grid onto
    clusters (MPAP_SEARCH_NO_GRID)."""
    B, rm, gold = bench_shard
    beta = _betas(gold)[0]
    monkeypatch.setenv("MPAP_SEARCH_CTA", "1")
    before = mp.mpap_search_launches()
    paths, res = B.search(rm, [beta] * len(B.probs), path_capacity=512)
    assert mp.mpap_search_launches()["cta"] > before["cta"]
    for q, gd in enumerate(gold["envs"]):
        _check(res, paths, q, gd["searches"][0])
    monkeypatch.delenv("MPAP_SEARCH_CTA")
    monkeypatch.setenv("MPAP_SEARCH_NO_GRID", "1")
    envs = np.arange(8, dtype=np.int32) * 7
    before = mp.mpap_search_launches()
    paths, res = B.search(rm, [beta] * 8, path_capacity=512, envs=envs)
    after = mp.mpap_search_launches()
    assert after["cluster"] > before["cluster"] and after["grid"] == before["grid"]
    for q, e in enumerate(envs):
        _check(res, paths, q, gold["envs"][e]["searches"][0])


def test_bench_shard_grid_single_queries(mp, bench_shard):
    """A batch of at most 8 queries runs query by query on the whole grid
    (cooperative launch), per-wave counters included."""
    B, rm, gold = bench_shard
    betas = _betas(gold)
    envs = np.array([3, 11, 29, 40, 63], dtype=np.int32)
    bq = [betas[k % len(betas)] for k in range(len(envs))]
    before = mp.mpap_search_launches()
    paths, res, wc = B.search(rm, bq, path_capacity=512, envs=envs, trace_waves=256)
    after = mp.mpap_search_launches()
    assert after["grid"] - before["grid"] >= len(envs) and after["cta"] == before["cta"]
    for q, e in enumerate(envs):
        _check(res, paths, q, gold["envs"][e]["searches"][q % len(betas)], counters=wc)


@pytest.mark.parametrize("name", ["c3", "c4"])
def test_full_csr_digests_single(mp, name):
    gold = json.load(open(os.path.join(GOLDEN, f"{name}_full.json")))
    prob = make_problem(load_config(name))
    rm = mp.pb.build_problem(prob)
    assert _digests(mp, rm, 0) == gold["digests"]
    rm.free()


def test_full_csr_digests_c5_golden_envs(mp):
    gold = json.load(open(os.path.join(GOLDEN, "c5_full.json")))["envs"]
    cfg = load_config("c5")
    B = mp.pb.Batch([make_problem(cfg, env_index=k) for k in range(len(gold))])
    rm = B.build()
    for e, gd in enumerate(gold):
        assert _digests(mp, rm, e) == gd["digests"], e
    rm.free()


@pytest.mark.parametrize("hints", ["process", "none"])
def test_c4_tightest_bound_single_query(mp, monkeypatch, hints):
    """C4 at 1.02 beta_min (the tightest bound of BASELINE.json configs[3]'s
    sweep): 105 waves, 2.1e8 relaxations, staircases of thousands of plans,
    so the CTA-cooperative and warp binary-search merges of large nodes run;
    whole result and every per-wave counter vs the oracle's stored run.
    With hints="none" (MPAP_SEARCH_NO_HINT) the fresh roadmap starts at the
    default capacities, so the overflow -> regrow -> rerun path runs too."""
    if hints == "none":
        monkeypatch.setenv("MPAP_SEARCH_NO_HINT", "1")
    path = os.path.join(GOLDEN, "c4_tight.json")
    if not os.path.exists(path):
        pytest.skip("tests/golden/c4_tight.json not generated")
    gold = json.load(open(path))
    prob = make_problem(load_config("c4"))
    rm = mp.pb.build_problem(prob)
    assert _digests(mp, rm, 0) == gold["digests"]
    for s in gold["searches"]:
        g = mp.pb.search_problem(rm, prob, float(s["beta"]), trace_waves=4096)
        assert g["status"] == s["status"] and g["waves"] == s["waves"]
        assert g["relaxations"] == s["relaxations"] and g["labels_inserted"] == s["labels_inserted"]
        assert g["wave_counters"].tolist() == s["wave_counters"]
        assert g["path"].tolist() == s["path"]
        assert _hex(g["cost"]) == s["cost"] and _hex(g["h"]) == s["h"] and _hex(g["h_peak"]) == s["h_peak"]
        if hints == "none":
            assert g["retries"] >= 1   # thousands of plans per node overflow the default staircase capacity
    rm.free()


def test_all_512_c5_queries_on_one_gpu(mp):
    """BASELINE.json configs[4] whole: the 512 C5 environments built as one
    batch and searched as one 512-query batch (one CTA per query) on one GPU
    -- the strong-scaling base of bench.py --queries-per-gpu 512 -- every
    result vs the oracle's stored run (c5_all.json), CSR digests of 16
    sampled environments."""
    gold = json.load(open(os.path.join(GOLDEN, "c5_all.json")))
    cfg = load_config("c5")
    assert len(gold["envs"]) == int(cfg["n_queries"]) and gold["beta"] == float(cfg["betas"][1])
    B = mp.pb.Batch([make_problem(cfg, env_index=k) for k in range(len(gold["envs"]))])
    rm = B.build()
    before = mp.mpap_search_launches()
    paths, res = B.search(rm, [gold["beta"]] * len(gold["envs"]), path_capacity=512)
    assert mp.mpap_search_launches()["cta"] > before["cta"]
    for q, gd in enumerate(gold["envs"]):
        _check(res, paths, q, gd["searches"][0])
    for e in range(0, len(gold["envs"]), 32):
        assert _digests(mp, rm, e) == gold["envs"][e]["digests"], e
    rm.free()
