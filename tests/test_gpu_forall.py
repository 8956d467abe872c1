"""GPU parity for NEXT-3: the per-edge peak summaries
(S, C) written by k_heuristic and the MPAP_SEARCH_FORALL_T cutoff of Eq. 2
(reading R11) against the oracle (orc_build_peaks, orc_search_ex)."""
import numpy as np
import pytest

from synth import load_config, make_problem
from test_gpu_parity import assert_search_equal, bits, mp, small  # noqa: F401  (mp is a fixture)

pytestmark = pytest.mark.gpu
INF = float("inf")


@pytest.mark.parametrize("name,n", [("c1", None), ("c2", None), ("c3", 400), ("c3", 2)])
def test_peaks_bit_exact(mp, orc, name, n):
    prob = small(name, n)
    rm = mp.pb.build_problem(prob, edge_peaks=True)
    orm = orc.build_roadmap(prob)
    S, Cp = mp.mpap_roadmap_export_peaks(rm)
    oS, oC = orc.build_peaks(prob, orm)
    assert np.array_equal(bits(S), bits(oS))
    assert np.array_equal(bits(Cp), bits(oC))
    g = mp.mpap_roadmap_export(rm)
    free = g["coll"] == 0
    assert (S[~free] == 0).all() and (Cp[~free] == 0).all()
    assert (S[free] >= np.maximum(g["s"][free], 0)).all() and (Cp[free] >= g["c"][free]).all()


@pytest.mark.parametrize("name", ["c1", "c2"])
def test_forall_search_parity(mp, orc, name):
    prob = make_problem(load_config(name))
    rm = mp.pb.build_problem(prob, edge_peaks=True)
    orm = orc.build_roadmap(prob)
    for beta in prob.betas:
        g = mp.pb.search_problem(rm, prob, beta, trace_waves=4096, forall_t=True)
        o = orc.search(orm, prob, beta, forall_t=True)
        assert_search_equal(g, o)


def test_forall_search_parity_c3_reduced(mp, orc):
    prob = small("c3", 700)
    rm = mp.pb.build_problem(prob, edge_peaks=True)
    orm = orc.build_roadmap(prob)
    for beta in [INF, 6.0, 3.0, 2.0]:
        g = mp.pb.search_problem(rm, prob, beta, trace_waves=4096, forall_t=True)
        assert_search_equal(g, orc.search(orm, prob, beta, forall_t=True))


def test_forall_batch_equals_single(mp, orc):
    prob = small("c3", 700)
    rm = mp.pb.build_problem(prob, edge_peaks=True)
    betas = [INF, 6.0, 3.0, 2.0, 1.0]
    paths, res = mp.pb.beta_sweep(rm, prob, betas, forall_t=True)
    for k, beta in enumerate(betas):
        g = mp.pb.search_problem(rm, prob, beta, forall_t=True)
        assert int(res[k]["status"]) == g["status"]
        if g["status"] == 0:
            assert paths[k][: res[k]["path_len"]].tolist() == g["path"].tolist()
            assert bits(np.float32(res[k]["cost"])) == bits(np.float32(g["cost"]))


def _peak_import(mp, orc, rng, n, deg):
    """Random CSR whose edge data come from increment sequences (oracle folds)."""
    rows, incs = [], []
    for u in range(n):
        for v in rng.choice([x for x in range(n) if x != u], size=min(deg, n - 1), replace=False):
            inc = (rng.integers(-16, 24, int(rng.integers(1, 6))) / 64.0)
            rows.append((u, int(v), float(rng.uniform(0.1, 1.0)), int(rng.random() < 0.1)))
            incs.append(inc)
    order = sorted(range(len(rows)), key=lambda k: (rows[k][0], rows[k][1]))
    rows = [rows[k] for k in order]
    incs = [incs[k] for k in order]
    row_ptr = np.zeros(n + 1, np.int32)
    for (u, _, _, _) in rows:
        row_ptr[u + 1] += 1
    row_ptr = np.cumsum(row_ptr).astype(np.int32)
    dst = np.array([r[1] for r in rows], np.int32)
    coll = np.array([r[3] for r in rows], np.uint8)
    w = np.array([r[2] for r in rows], np.float32)
    s = np.zeros(len(rows), np.float32)
    c = np.zeros(len(rows), np.float32)
    S = np.zeros(len(rows), np.float32)
    Cp = np.zeros(len(rows), np.float32)
    for k, inc in enumerate(incs):
        if not coll[k]:
            s[k], c[k] = orc.fold_summary(inc)
            S[k], Cp[k] = orc.fold_peak(inc)
    pos = np.zeros((n, 2))
    pos[:, 0] = np.arange(n)
    dc = dst.astype(np.uint32) | (coll.astype(np.uint32) << 31)
    rm = mp.mpap_roadmap_import(pos, row_ptr, dc, w, s, c, 1.0)
    return rm, dict(n=n, row_ptr=row_ptr, dst=dst, coll=coll, w=w, s=s, c=c, S=S, C=Cp)


@pytest.mark.parametrize("seed", range(8))
def test_forall_random_imported_graphs(mp, orc, seed):
    rng = np.random.default_rng(1300 + seed)
    n = int(rng.integers(5, 50))
    rm, g = _peak_import(mp, orc, rng, n, int(rng.integers(2, 6)))
    with pytest.raises(mp.MpapError) as ei:   # no peaks attached yet
        mp.mpap_search(rm, 0, 0, [n - 1.25, -0.5], [n - 0.75, 0.5], INF, 0.5, forall_t=True)
    assert ei.value.status == mp.MPAP_ERR_INVALID_ARGUMENT
    mp.mpap_roadmap_set_peaks(rm, g["S"], g["C"])
    S, Cp = mp.mpap_roadmap_export_peaks(rm)
    assert np.array_equal(bits(S), bits(g["S"])) and np.array_equal(bits(Cp), bits(g["C"]))
    goal = np.zeros(n, np.uint8)
    goal[n - 1] = 1
    for lam in [0.5, 0.1]:
        for beta in [INF, 1.0, 0.6, 0.4]:
            gr = mp.mpap_search(rm, 0, 0, [n - 1.25, -0.5], [n - 0.75, 0.5], beta, lam, trace_waves=4096,
                                forall_t=True)
            o = orc.search_csr(n, g["row_ptr"], g["dst"], g["coll"], g["w"], g["s"], g["c"], goal, 0, beta, lam, 1.0,
                               S=g["S"], Cp=g["C"], forall_t=True)
            assert_search_equal(gr, o)


def test_forall_needs_peaks(mp):
    """A roadmap built without edge_peaks carries no peaks: the all-t search
    and the peak export are INVALID_ARGUMENT, the node-only search runs."""
    prob = small("c2", 60)
    rm = mp.pb.build_problem(prob)
    for call in (lambda: mp.pb.search_problem(rm, prob, INF, forall_t=True),
                 lambda: mp.mpap_roadmap_export_peaks(rm),
                 lambda: mp.pb.beta_sweep(rm, prob, [INF], forall_t=True)):
        with pytest.raises(mp.MpapError) as ei:
            call()
        assert ei.value.status == mp.MPAP_ERR_INVALID_ARGUMENT
    assert mp.pb.search_problem(rm, prob, INF)["status"] in (0, 3)
