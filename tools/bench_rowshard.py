"""Row-sharded roadmap build of one large environment (C4,
n = 16 001) across the ranks of one node: rank g builds rows
[g n/G, (g+1) n/G) (mpap_build_roadmap_rows), the CSR blocks are all-gathered
once (NCCL) and concatenated, and every rank imports the full CSR and runs
the query.  Times: the block build (CUDA events, max over ranks), the
gather + assembly + import, and the search; the plan is checked against a
full single-GPU build on rank 0.

    python tools/bench_rowshard.py                       # G = 1
    python -m torch.distributed.run --nproc-per-node G --master-addr 127.0.0.1 tools/bench_rowshard.py
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import build_ext
    if rank == 0:
        build_ext.build()
    if world > 1:
        dist.barrier()
    import paper_1705_02408_b200 as mp
    from paper_1705_02408_b200 import dist as md
    from paper_1705_02408_b200.problem import build_problem, build_problem_rows, search_problem
    from synth import load_config, make_problem
    cfg = load_config(os.environ.get("MPAP_ROWSHARD_CONFIG", "c4"))
    prob = make_problem(cfg)
    beta = float(cfg["betas"][1])
    b, e = md.row_block(rank, world, prob.n)
    build_problem_rows(prob, b, e).free()   # warm-up
    torch.cuda.synchronize()
    reps = 3
    t_build, t_asm, t_search = [], [], []
    for _ in range(reps):
        if world > 1:
            dist.barrier()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        ev[0].record()
        part = build_problem_rows(prob, b, e)
        ev[1].record()
        ev[1].synchronize()
        t_build.append(ev[0].elapsed_time(ev[1]))
        h0 = time.perf_counter()
        block = md.csr_block(mp.mpap_roadmap_export(part), b, e)
        part.free()
        full = md.assemble_csr(md.gather_csr_blocks(block, world), prob.n)
        rm = mp.mpap_roadmap_import(prob.samples[:, : prob.pos_dim], full["row_ptr"], full["dst_coll"], full["w"],
                                    full["s"], full["c"], prob.r)
        t_asm.append((time.perf_counter() - h0) * 1e3)
        h1 = time.perf_counter()
        res = search_problem(rm, prob, beta)
        t_search.append((time.perf_counter() - h1) * 1e3)
        rm.free()
    tb = torch.tensor([float(np.median(t_build))], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(tb, op=dist.ReduceOp.MAX)
    out = {"config": cfg["name"], "n": prob.n, "world": world, "block_build_ms_max_over_ranks": float(tb.item()),
           "gather_assemble_import_ms": float(np.median(t_asm)), "search_ms": float(np.median(t_search)),
           "status": int(res["status"]), "cost": float(res["cost"])}
    # one GPU: time every block of a G-way split alone (the per-rank build
    # time a G-rank run would see, without the gather); not a multi-GPU number
    if world == 1:
        per = {}
        for G in (2, 4, 8):
            ts = []
            for g in range(G):
                bb, ee = md.row_block(g, G, prob.n)
                ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
                ev[0].record()
                part = build_problem_rows(prob, bb, ee)
                ev[1].record()
                ev[1].synchronize()
                ts.append(ev[0].elapsed_time(ev[1]))
                part.free()
            per[str(G)] = {"max_block_ms": max(ts), "blocks_ms": [round(t, 3) for t in ts]}
        out["one_gpu_block_times"] = per
    if rank == 0:
        ref_rm = build_problem(prob)
        ref = search_problem(ref_rm, prob, beta)
        ref_rm.free()
        out["same_plan_as_single_gpu_build"] = bool(ref["path"].tolist() == res["path"].tolist())
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
