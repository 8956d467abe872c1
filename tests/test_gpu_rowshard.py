"""GPU parity of the row-sharded roadmap build (Alg. 2 is
"embarrassingly parallel" over rows): mpap_build_roadmap_rows builds
row blocks; their exported CSRs concatenated in row order equal the
single-GPU build bit for bit, and a search on the assembled (imported)
roadmap equals the search on the full build.  The blocks are built one after
the other on one GPU here (nothing waits on anything); the multi-rank
gather/assembly logic is covered by tests/test_dist.py (gloo, world 2)."""
import numpy as np
import pytest

from synth import load_config, make_problem

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mp():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import build_ext
    build_ext.build()
    import paper_1705_02408_b200 as m
    import paper_1705_02408_b200.problem as pb
    import paper_1705_02408_b200.dist as dist
    m.pb = pb
    m.dist = dist
    return m


@pytest.mark.parametrize("name,n,world", [("c1", 500, 2), ("c3", 1500, 3), ("c4", 16000, 4)])
def test_row_blocks_assemble_to_full_build(mp, name, n, world):
    cfg = load_config(name)
    cfg["n_samples"] = n
    prob = make_problem(cfg)
    full_rm = mp.pb.build_problem(prob)
    full = mp.mpap_roadmap_export(full_rm)
    blocks = []
    for rank in range(world):
        b, e = mp.dist.row_block(rank, world, prob.n)
        part = mp.pb.build_problem_rows(prob, b, e)
        ex = mp.mpap_roadmap_export(part)
        rp = ex["row_ptr"]
        assert np.all(np.diff(rp)[:b] == 0) and np.all(np.diff(rp)[e:] == 0)   # only its rows have edges
        blocks.append(mp.dist.csr_block(ex, b, e))
        part.free()
    asm = mp.dist.assemble_csr(blocks, prob.n)
    assert np.array_equal(asm["row_ptr"], full["row_ptr"])
    assert np.array_equal(asm["dst_coll"] & 0x7FFFFFFF, full["dst"].astype(np.uint32))
    assert np.array_equal(asm["dst_coll"] >> 31, full["coll"].astype(np.uint32))
    for k in ("w", "s", "c"):
        assert np.array_equal(asm[k].view(np.uint32), full[k].view(np.uint32)), k
    imp = mp.mpap_roadmap_import(prob.samples[:, : prob.pos_dim], asm["row_ptr"], asm["dst_coll"], asm["w"],
                                 asm["s"], asm["c"], prob.r)
    for beta in [float(b) for b in cfg["betas"][:2]]:
        a = mp.pb.search_problem(imp, prob, beta)
        f = mp.pb.search_problem(full_rm, prob, beta)
        assert a["status"] == f["status"] and a["path"].tolist() == f["path"].tolist()
        assert np.float32(a["cost"]) == np.float32(f["cost"]) and np.float32(a["h"]) == np.float32(f["h"])
    imp.free()
    full_rm.free()


def test_row_range_validation(mp):
    prob = make_problem(load_config("c1"))
    with pytest.raises(mp.MpapError):
        mp.pb.build_problem_rows(prob, 10, 5)
    with pytest.raises(mp.MpapError):
        mp.pb.build_problem_rows(prob, 0, prob.n + 1)
    empty = mp.pb.build_problem_rows(prob, 7, 7)
    assert mp.mpap_roadmap_info(empty)["nnz"] == 0
    empty.free()
