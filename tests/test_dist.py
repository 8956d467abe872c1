"""World-size-2 gloo test of the multi-GPU path's host logic:
disjoint weak-scaling shards and the all-gather of 48-byte result records in
rank order.  Runs on CPU; the GPU run uses NCCL through the same function."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as tmp

RESULT_DTYPE = np.dtype([("status", np.int32), ("path_len", np.int32), ("waves", np.int32), ("retries", np.int32),
                         ("cost", np.float32), ("h", np.float32), ("h_peak", np.float32), ("pad", np.float32),
                         ("relaxations", np.int64), ("labels_inserted", np.int64)])


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, Q, outdir):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch
    import torch.distributed as dist
    # import the submodule without loading libmpap.so (no GPU library needed here)
    import importlib.util
    spec = importlib.util.spec_from_file_location(
        "mpap_dist", os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                  "paper_1705_02408_b200", "dist.py"))
    md = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(md)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    envs = md.shard_envs(rank, world, Q)
    rec = np.zeros(Q, dtype=RESULT_DTYPE)
    rec["status"] = 0
    rec["path_len"] = np.array(envs) + 1
    rec["cost"] = np.array(envs, dtype=np.float32) * 0.5
    rec["relaxations"] = np.array(envs) * 1000
    local = torch.from_numpy(rec.view(np.uint8).copy())
    out = md.gather_results(local, world)
    got = md.records(out, RESULT_DTYPE)
    np.save(os.path.join(outdir, f"r{rank}.npy"), got)
    dist.destroy_process_group()


def _mc_worker(rank, world, port, trials, outdir):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch
    import torch.distributed as dist
    import importlib.util
    spec = importlib.util.spec_from_file_location(
        "mpap_dist", os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                  "paper_1705_02408_b200", "dist.py"))
    md = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(md)
    import oracle
    from synth import line_problem, mc_params
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    prob = line_problem([(0.0, 0.0, 1.5, 0.0, 0.0, 0.0, 1.0, 0.0), (3.0, 0.0, 1.5, 0.0, 0.0, 0.0, 1.0, 0.0)],
                        features=[[1.5, 3.0, 1.5]])
    mc = mc_params(trials=trials, sigma_imu=0.5, sigma_vis=0.2, delta=0.05)
    t0, n = md.mc_trial_shard(rank, world, trials)
    # the oracle stands in for this rank's k_mc launch (CPU test of the host logic)
    r = oracle.mc_verify(prob, [0, 1], mc, t0, n)
    cnt = md.reduce_exceed(torch.tensor([r["exceed"]], dtype=torch.int64))
    np.save(os.path.join(outdir, f"mc{rank}.npy"), np.array([int(cnt[0]), t0, n]))
    dist.destroy_process_group()


def test_mc_sharded_trials_two_ranks(tmp_path, orc):
    """Sharded Monte Carlo (NEXT-4): trials split across 2 ranks, one
    all-reduce of the exceedance count equals the single-process count."""
    world, trials = 2, 41
    port = _free_port()
    tmp.start_processes(_mc_worker, args=(world, port, trials, str(tmp_path)), nprocs=world, start_method="spawn")
    a = np.load(tmp_path / "mc0.npy")
    b = np.load(tmp_path / "mc1.npy")
    from synth import line_problem, mc_params
    prob = line_problem([(0.0, 0.0, 1.5, 0.0, 0.0, 0.0, 1.0, 0.0), (3.0, 0.0, 1.5, 0.0, 0.0, 0.0, 1.0, 0.0)],
                        features=[[1.5, 3.0, 1.5]])
    full = orc.mc_verify(prob, [0, 1], mc_params(trials=trials, sigma_imu=0.5, sigma_vis=0.2, delta=0.05))
    assert a[0] == b[0] == full["exceed"]
    assert a[1] == 0 and b[1] == a[2] and a[2] + b[2] == trials


def _csr_worker(rank, world, port, outdir):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch.distributed as dist
    import importlib.util
    spec = importlib.util.spec_from_file_location(
        "mpap_dist", os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                  "paper_1705_02408_b200", "dist.py"))
    md = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(md)
    import oracle
    from synth import load_config, make_problem
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = load_config("c1")
    cfg["n_samples"] = 150
    prob = make_problem(cfg)
    b, e = md.row_block(rank, world, prob.n)
    # this rank's row block (the oracle's rows stand in for k_near/k_edges on the rank's GPU)
    rows = [oracle.build_row(prob, u) for u in range(b, e)]
    block = {"b": b, "e": e, "counts": np.array([r["dst"].size for r in rows], np.int32),
             "dst_coll": np.concatenate([r["dst"].astype(np.uint32) | (r["coll"].astype(np.uint32) << np.uint32(31))
                                         for r in rows]),
             "w": np.concatenate([r["w"] for r in rows]), "s": np.concatenate([r["s"] for r in rows]),
             "c": np.concatenate([r["c"] for r in rows])}
    full = md.assemble_csr(md.gather_csr_blocks(block, world), prob.n)
    np.savez(os.path.join(outdir, f"csr{rank}.npz"), **full)
    dist.destroy_process_group()


def test_row_sharded_csr_two_ranks(tmp_path, orc):
    """Row-sharded build: the all-gathered, concatenated
    row blocks equal the single-process CSR bit for bit on every rank."""
    world = 2
    port = _free_port()
    tmp.start_processes(_csr_worker, args=(world, port, str(tmp_path)), nprocs=world, start_method="spawn")
    from synth import load_config, make_problem
    cfg = load_config("c1")
    cfg["n_samples"] = 150
    o = orc.build_roadmap(make_problem(cfg))
    for rank in range(world):
        g = np.load(tmp_path / f"csr{rank}.npz")
        assert np.array_equal(g["row_ptr"], o["row_ptr"])
        assert np.array_equal(g["dst_coll"] & 0x7FFFFFFF, o["dst"].astype(np.uint32))
        assert np.array_equal(g["dst_coll"] >> 31, o["coll"].astype(np.uint32))
        for k in ("w", "s", "c"):
            assert np.array_equal(g[k].view(np.uint32), o[k].view(np.uint32)), k


def test_gather_two_ranks(tmp_path):
    world, Q = 2, 5
    port = _free_port()
    tmp.start_processes(_worker, args=(world, port, Q, str(tmp_path)), nprocs=world, start_method="spawn")
    a = np.load(tmp_path / "r0.npy")
    b = np.load(tmp_path / "r1.npy")
    assert np.array_equal(a, b)
    assert a["path_len"].tolist() == list(range(1, world * Q + 1))
    assert a["relaxations"].tolist() == [1000 * k for k in range(world * Q)]


def test_shards_disjoint_and_cover():
    import importlib.util
    spec = importlib.util.spec_from_file_location(
        "mpap_dist", os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                  "paper_1705_02408_b200", "dist.py"))
    md = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(md)
    for world in (1, 2, 4, 8):
        all_envs = sum((md.shard_envs(r, world, 64) for r in range(world)), [])
        assert sorted(all_envs) == list(range(64 * world))
    with pytest.raises(ValueError):
        md.shard_envs(2, 2, 4)
    for world in (1, 2, 3, 8):
        for n in (0, 1, 5, 4001):
            blocks = [md.row_block(r, world, n) for r in range(world)]
            assert blocks[0][0] == 0 and blocks[-1][1] == n
            assert all(blocks[r][1] == blocks[r + 1][0] for r in range(world - 1))
        for trials in (0, 1, 7, 1000):
            parts = [md.mc_trial_shard(r, world, trials) for r in range(world)]
            assert sum(n for _, n in parts) == trials
            assert all(parts[r][0] + parts[r][1] == parts[r + 1][0] for r in range(world - 1))


def test_bench_launcher_spawns_ranks():
    """bench.py --gpus 2 outside torchrun re-launches itself as 2 ranks
    (torch.distributed.run, 127.0.0.1 rendezvous); the ranks gather their
    shards' result records with the bench's collective and reduce the time
    MAX over ranks; rank 0 alone prints one JSON line (gloo on CPU)."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--launcher-selftest",
                          "--queries-per-gpu", "3"], capture_output=True, text=True, timeout=300, env=env, cwd=root)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["gathered_queries"] == 6 and d["records_in_rank_order"]
    assert d["max_over_ranks"] == 2.0
