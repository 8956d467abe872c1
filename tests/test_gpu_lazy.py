"""GPU parity of lazy edge evaluation (NEXT-1 part i; "the number of
new edge collision checks can be limited", P:407 the heuristic is 65 % of the
time): a roadmap built with ``lazy_edges`` holds Near + Cost only; the
single-query search evaluates a row's collision bits and heuristic summaries
when it first expands a plan at that node (suspend / evaluate / resume).

Bar: the lazy search returns the eager search's result bit for bit (status,
path, cost, h, h_peak, waves, relaxations, inserted, per-wave counters), the
eager result equals the oracle, and once every row is evaluated the CSR equals
the eager build bit for bit.
"""
import numpy as np
import pytest

from synth import load_config, make_problem

pytestmark = pytest.mark.gpu
INF = float("inf")


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


def same(a, b):
    assert a["status"] == b["status"]
    for k in ("waves", "relaxations", "labels_inserted"):
        assert a[k] == b[k], k
    assert a["path"].tolist() == b["path"].tolist()
    for k in ("cost", "h", "h_peak"):
        assert np.float32(a[k]).view(np.uint32) == np.float32(b[k]).view(np.uint32), k


def small(name, n):
    cfg = load_config(name)
    cfg["n_samples"] = n
    return make_problem(cfg)


@pytest.mark.parametrize("name,n,betas", [("c1", 500, [INF, 0.2174]), ("c2", 600, [INF, 1.1762]),
                                          ("c3", 1200, [INF, 2.6876, 2.1931])])
def test_lazy_search_equals_eager(mp, name, n, betas):
    prob = small(name, n)
    eager = mp.pb.build_problem(prob)
    for beta in betas:
        lazy = mp.pb.build_problem(prob, lazy_edges=True)
        assert mp.mpap_roadmap_rows_evaluated(lazy) == 0
        gl = mp.pb.search_problem(lazy, prob, beta, trace_waves=256)
        ge = mp.pb.search_problem(eager, prob, beta, trace_waves=256)
        same(gl, ge)
        assert np.array_equal(gl["wave_counters"], ge["wave_counters"])
        rows = mp.mpap_roadmap_rows_evaluated(lazy)
        assert 0 < rows <= prob.n
        # a second search on the same lazy roadmap reuses the evaluated rows
        same(mp.pb.search_problem(lazy, prob, beta), ge)
        lazy.free()
    eager.free()


def test_lazy_equals_oracle_and_full_export(mp, orc):
    prob = small("c3", 700)
    lazy = mp.pb.build_problem(prob, lazy_edges=True)
    o = orc.build_roadmap(prob)
    for beta in (INF, 2.6876):
        g = mp.pb.search_problem(lazy, prob, beta)
        r = orc.search(o, prob, beta)
        assert g["status"] == r["status"]
        if r["status"] == 0:
            assert g["path"].tolist() == r["path"].tolist()
            assert np.float32(g["cost"]) == r["cost"] and np.float32(g["h"]) == r["h"]
    # export evaluates the remaining rows: the CSR is the eager (= oracle) one
    ex = mp.mpap_roadmap_export(lazy)
    assert mp.mpap_roadmap_rows_evaluated(lazy) == prob.n
    for k in ("row_ptr", "dst", "coll"):
        assert np.array_equal(ex[k], o[k]), k
    for k in ("w", "s", "c"):
        assert np.array_equal(ex[k].view(np.uint32), o[k].view(np.uint32)), k
    assert mp.mpap_roadmap_info(lazy)["nnz_free"] == int((o["coll"] == 0).sum())
    lazy.free()


def test_lazy_beta_sweep_equals_eager(mp):
    prob = small("c3", 600)
    lazy = mp.pb.build_problem(prob, lazy_edges=True)
    eager = mp.pb.build_problem(prob)
    betas = [INF, 2.6876, 2.1931]
    pl, rl = mp.pb.beta_sweep(lazy, prob, betas)
    pe, re_ = mp.pb.beta_sweep(eager, prob, betas)
    assert np.array_equal(rl, re_)
    for k in range(len(betas)):   # path rows beyond path_len are unspecified (mpap.h)
        assert np.array_equal(pl[k][: rl["path_len"][k]], pe[k][: re_["path_len"][k]])
    assert 0 < mp.mpap_roadmap_rows_evaluated(lazy) <= prob.n
    lazy.free()
    eager.free()


def test_lazy_batch_of_envs_equals_eager(mp):
    """A lazy multi-environment batch (the bench's C5 shape, 8 full-size
    environments): the batched search suspends per wave, the library
    evaluates the union of requested rows and resumes; results equal the
    eager batch record for record."""
    cfg = load_config("c5")
    probs = [make_problem(cfg, env_index=k) for k in range(8)]
    B = mp.pb.Batch(probs)
    eager = B.build()
    pe, re_ = B.search(eager, [float(cfg["betas"][1])] * len(probs))
    B.prm.lazy_edges = 1
    lazy = B.build()
    B.prm.lazy_edges = 0
    pl, rl = B.search(lazy, [float(cfg["betas"][1])] * len(probs))
    for k in ("status", "path_len", "waves", "cost", "h", "h_peak", "relaxations", "labels_inserted"):
        assert np.array_equal(rl[k], re_[k]), k
    for k in range(len(probs)):   # path rows beyond path_len are unspecified (mpap.h)
        assert np.array_equal(pl[k][: rl["path_len"][k]], pe[k][: re_["path_len"][k]])
    rows = sum(mp.mpap_roadmap_rows_evaluated(lazy, e) for e in range(len(probs)))
    assert 0 < rows < sum(p.n for p in probs)
    lazy.free()
    eager.free()


def test_lazy_forall_t_equals_eager(mp):
    """Lazy roadmap built with edge peaks: the Eq. 2 for-all-t search (NEXT-3)
    reads peaks evaluated on demand and equals the eager one."""
    prob = small("c3", 700)
    eager = mp.pb.build_problem(prob, edge_peaks=True)
    lazy = mp.pb.build_problem(prob, edge_peaks=True, lazy_edges=True)
    for beta in (2.6876, 2.1931):
        same(mp.pb.search_problem(lazy, prob, beta, forall_t=True),
             mp.pb.search_problem(eager, prob, beta, forall_t=True))
    Sl, Cl = mp.mpap_roadmap_export_peaks(lazy)
    Se, Ce = mp.mpap_roadmap_export_peaks(eager)
    assert np.array_equal(Sl.view(np.uint32), Se.view(np.uint32)) and np.array_equal(Cl.view(np.uint32),
                                                                                      Ce.view(np.uint32))
    lazy.free()
    eager.free()


def test_lazy_c4_full_single_query(mp):
    """C4 at full size: the whole-grid lazy search equals the eager one at the
    agnostic bound and at 2 beta_min (39 waves of suspend / evaluate / resume)."""
    cfg = load_config("c4")
    prob = make_problem(cfg)
    eager = mp.pb.build_problem(prob)
    for beta in (INF, 17.303):
        lazy = mp.pb.build_problem(prob, lazy_edges=True)
        same(mp.pb.search_problem(lazy, prob, beta), mp.pb.search_problem(eager, prob, beta))
        assert mp.mpap_roadmap_rows_evaluated(lazy) < prob.n
        lazy.free()
    eager.free()
