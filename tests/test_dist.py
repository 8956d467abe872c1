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
