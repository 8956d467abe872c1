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


@pytest.mark.parametrize("world", [1, 2, 3, 5])
def test_device_blocks_assemble_to_full_c4(mp, world):
    """The device path (mpap_roadmap_block_device per rank, the slots stacked
    as NCCL's all_gather_into_tensor lays them out, mpap_roadmap_assemble_device)
    gives the full C4 CSR bit for bit (digests of tests/golden/c4_full.json,
    oracle only) and the same search."""
    import json
    import os
    import sys
    import torch
    golden = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
    sys.path.insert(0, golden)
    from digest import csr_digests
    gold = json.load(open(os.path.join(golden, "c4_full.json")))
    prob = make_problem(load_config("c4"))
    dev = torch.device("cuda")
    parts, sizes = [], []
    for rank in range(world):
        b, e = mp.dist.row_block(rank, world, prob.n)
        part = mp.pb.build_problem_rows(prob, b, e)
        sizes.append((e - b, mp.mpap_roadmap_info(part)["nnz"]))
        parts.append(part)
    rows_max = max(s[0] for s in sizes)
    nnz_max = max(max(s[1] for s in sizes), 1)
    gc = torch.zeros((world, rows_max), dtype=torch.int32, device=dev)
    ge = torch.zeros((world, nnz_max, 4), dtype=torch.int32, device=dev)
    for rank, part in enumerate(parts):
        assert mp.mpap_roadmap_block_device(part, gc[rank], ge[rank]) == sizes[rank][1]
        part.free()
    row_begin = [mp.dist.row_block(g, world, prob.n)[0] for g in range(world)] + [prob.n]
    rm = mp.mpap_roadmap_assemble_device(prob.samples[:, :3], row_begin, gc, ge, prob.r)
    assert csr_digests(mp.mpap_roadmap_export(rm)) == gold["digests"]
    assert mp.mpap_roadmap_info(rm)["nnz_free"] == gold["nnz_free"]
    s = gold["searches"][1]
    g = mp.pb.search_problem(rm, prob, float(s["beta"]), trace_waves=4096)
    assert g["path"].tolist() == s["path"] and g["wave_counters"].tolist() == s["wave_counters"]
    rm.free()


def test_device_assemble_rejects_bad_blocks(mp):
    import torch
    dev = torch.device("cuda")
    pos = np.zeros((4, 2))
    gc = torch.tensor([[1, 1], [1, 0]], dtype=torch.int32, device=dev)
    ge = torch.zeros((2, 2, 4), dtype=torch.int32, device=dev)
    ge[0, 0, 0] = 1
    ge[0, 1, 0] = 9      # dst out of range
    ge[1, 0, 0] = 0
    with pytest.raises(mp.MpapError):
        mp.mpap_roadmap_assemble_device(pos, [0, 2, 4], gc, ge, 1.0)
    with pytest.raises(mp.MpapError):   # blocks do not tile [0, n)
        mp.mpap_roadmap_assemble_device(pos, [0, 2, 3], gc, ge, 1.0)
