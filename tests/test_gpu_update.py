"""GPU parity for NEXT-1: mpap_roadmap_update
re-evaluates only the edges a change of obstacles/features can affect, and the
updated roadmap equals the oracle's full build of the new environment bit for
bit (the plain definition an incremental update must meet)."""
import dataclasses

import numpy as np
import pytest

from test_gpu_parity import assert_roadmap_equal, assert_search_equal, bits, mp, small  # noqa: F401

pytestmark = pytest.mark.gpu
INF = float("inf")


def _changes(prob, rng):
    """A sequence of environment edits of the kinds an online map produces."""
    d = prob.pos_dim
    box0, feat0 = prob.obstacles.copy(), prob.features.copy()
    span = prob.ws_hi[:d] - prob.ws_lo[:d]
    seq = []
    b = box0.copy()
    b[0, :d] += 0.02 * span
    b[0, d:] += 0.02 * span
    seq.append(("move box", b, feat0))
    seq.append(("remove box", np.delete(b, 1, axis=0), feat0))
    lo = prob.ws_lo[:d] + 0.4 * span
    nb = np.concatenate([np.delete(b, 1, axis=0), np.concatenate([lo, lo + 0.05 * span])[None]])
    seq.append(("add box", nb, feat0))
    f = feat0.copy()
    f[:3] += 0.03 * span
    f = np.concatenate([np.delete(f, 5, axis=0), prob.ws_lo[:d] + rng.uniform(0, 1, (2, d)) * span])
    seq.append(("edit features", nb, f))
    seq.append(("no change (reordered)", nb[::-1].copy(), f[::-1].copy()))
    seq.append(("clear all", np.zeros((0, 2 * d)), np.zeros((0, d))))
    seq.append(("restore", box0, feat0))
    return seq


@pytest.mark.parametrize("name,n,peaks", [("c1", None, False), ("c2", 400, False), ("c3", 500, True),
                                          ("c4", 300, False)])
def test_update_equals_full_build(mp, orc, name, n, peaks):
    prob = small(name, n)
    rm = mp.pb.build_problem(prob, edge_peaks=peaks)
    nnz = mp.mpap_roadmap_info(rm)["nnz"]
    rng = np.random.default_rng(7)
    for what, boxes, feats in _changes(prob, rng):
        k = mp.mpap_roadmap_update(rm, 0, boxes, feats)
        newp = dataclasses.replace(prob, obstacles=np.ascontiguousarray(boxes),
                                   features=np.ascontiguousarray(feats))
        o = orc.build_roadmap(newp)
        assert_roadmap_equal(mp.mpap_roadmap_export(rm), o)
        info = mp.mpap_roadmap_info(rm)
        assert info["nnz_free"] == int((o["coll"] == 0).sum()), what
        assert 0 <= k <= nnz, what
        if what.startswith("no change"):
            assert k == 0
        if peaks:
            S, Cp = mp.mpap_roadmap_export_peaks(rm)
            oS, oC = orc.build_peaks(newp, o)
            assert np.array_equal(bits(S), bits(oS)) and np.array_equal(bits(Cp), bits(oC)), what


def test_update_is_local_and_search_follows(mp, orc):
    """C3 at BASELINE size: moving one box re-evaluates a small fraction of the
    edges; sampled rows equal the oracle's rows of the new environment and the
    search on the updated roadmap equals a search on a fresh build."""
    from synth import load_config, make_problem
    prob = make_problem(load_config("c3"))
    rm = mp.pb.build_problem(prob)
    nnz = mp.mpap_roadmap_info(rm)["nnz"]
    d = prob.pos_dim
    boxes = prob.obstacles.copy()
    boxes[3, :d] += 0.3
    boxes[3, d:] += 0.3
    k = mp.mpap_roadmap_update(rm, 0, boxes, prob.features)
    assert 0 < k < nnz // 2, (k, nnz)
    newp = dataclasses.replace(prob, obstacles=boxes)
    g = mp.mpap_roadmap_export(rm)
    fresh = mp.pb.build_problem(newp)
    f = mp.mpap_roadmap_export(fresh)
    for key in ("row_ptr", "dst", "coll"):
        assert np.array_equal(g[key], f[key])
    for key in ("w", "s", "c"):
        assert np.array_equal(bits(g[key]), bits(f[key]))
    rng = np.random.default_rng(3)
    for u in rng.choice(prob.n, 12, replace=False):
        o = orc.build_row(newp, int(u))
        a, b = g["row_ptr"][u], g["row_ptr"][u + 1]
        assert np.array_equal(g["coll"][a:b], o["coll"])
        for key in ("s", "c"):
            assert np.array_equal(bits(g[key][a:b]), bits(o[key]))
    for beta in [INF, prob.betas[1]]:
        assert_search_equal(mp.pb.search_problem(rm, newp, beta, trace_waves=8192),
                            mp.pb.search_problem(fresh, newp, beta, trace_waves=8192))


def test_update_one_env_of_a_batch(mp, orc):
    from paper_1705_02408_b200.problem import Batch
    probs = [small("c2", 300 + 50 * k) for k in range(3)]
    for k, p in enumerate(probs):
        p.samples = p.samples.copy()
    B = Batch(probs)
    rm = B.build()
    d = probs[1].pos_dim
    boxes = probs[1].obstacles.copy()
    boxes[:, :d] += 0.05
    boxes[:, d:] += 0.05
    mp.mpap_roadmap_update(rm, 1, boxes, probs[1].features[:10])
    newp = dataclasses.replace(probs[1], obstacles=boxes, features=probs[1].features[:10].copy())
    for env, p in enumerate([probs[0], newp, probs[2]]):
        assert_roadmap_equal(mp.mpap_roadmap_export(rm, env), orc.build_roadmap(p))


def test_update_rejects_bad_input(mp):
    prob = small("c2", 80)
    rm = mp.pb.build_problem(prob)
    d = prob.pos_dim
    bad = prob.obstacles.copy()
    bad[0, 0] = bad[0, d] + 1.0   # lo > hi
    for call in (lambda: mp.mpap_roadmap_update(rm, 1, prob.obstacles, prob.features),
                 lambda: mp.mpap_roadmap_update(rm, 0, bad, prob.features)):
        with pytest.raises(mp.MpapError) as ei:
            call()
        assert ei.value.status == mp.MPAP_ERR_INVALID_ARGUMENT
    from graphs import csr
    g = csr(2, [(0, 1, 0.5, 0.0, 0.0)])
    imp = mp.mpap_roadmap_import(np.zeros((2, 2)), g["row_ptr"], g["dst"].astype(np.uint32), g["w"], g["s"],
                                 g["c"], 1.0)
    with pytest.raises(mp.MpapError) as ei:
        mp.mpap_roadmap_update(imp, 0, np.zeros((0, 4)), np.zeros((0, 2)))
    assert ei.value.status == mp.MPAP_ERR_INVALID_ARGUMENT


def test_update_of_a_lazy_roadmap(mp, orc):
    """A partially evaluated lazy roadmap (NEXT-1 part i) that is then updated
    (part ii) equals the oracle's full build of the new environment."""
    prob = small("c3", 500)
    lazy = mp.pb.build_problem(prob, lazy_edges=True)
    mp.pb.search_problem(lazy, prob, INF)          # evaluates some rows only
    assert mp.mpap_roadmap_rows_evaluated(lazy) < prob.n
    rng = np.random.default_rng(5)
    name, boxes, feats = _changes(prob, rng)[0]
    mp.mpap_roadmap_update(lazy, 0, boxes, feats)
    new = dataclasses.replace(prob, obstacles=boxes, features=feats)
    assert_roadmap_equal(mp.mpap_roadmap_export(lazy), orc.build_roadmap(new))
    lazy.free()
