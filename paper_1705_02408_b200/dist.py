"""Multi-GPU plumbing: independent environment+query units
are sharded across ranks with no data-path collective; the only exchange is
one all-gather of the fixed-size 48-byte result records (mpap_result) per
batch, never inside the wave loop.  A large single roadmap is built
row-sharded (rank g builds rows [g n/G, (g+1) n/G), mpap_build_roadmap_rows)
and its CSR blocks are all-gathered once and concatenated in row order.
Monte Carlo trials of a plan shard with one all-reduce of the exceedance
counts.  torch.distributed with NCCL on GPUs (gloo on CPU for tests).
"""
from __future__ import annotations

from typing import List

import numpy as np


def shard_envs(rank: int, world: int, per_rank: int) -> List[int]:
    """Weak scaling: rank r owns env indices [r*Q, (r+1)*Q)."""
    if not (0 <= rank < world) or per_rank < 0:
        raise ValueError("bad rank/world/per_rank")
    return list(range(rank * per_rank, (rank + 1) * per_rank))


def gather_results(local, world: int):
    """All-gather a uint8 tensor of result records (equal size on every rank)
    into one tensor ordered by rank."""
    import torch
    import torch.distributed as dist
    if world == 1:
        return local
    if dist.get_backend() == "nccl":
        out = torch.empty(world * local.numel(), dtype=local.dtype, device=local.device)
        dist.all_gather_into_tensor(out, local)
        return out
    parts = [torch.empty_like(local) for _ in range(world)]
    dist.all_gather(parts, local)
    return torch.cat(parts)


def records(tensor, dtype) -> np.ndarray:
    """View gathered bytes as structured result records."""
    return tensor.cpu().numpy().view(dtype)


def mc_trial_shard(rank: int, world: int, trials: int):
    """Monte Carlo trials of one plan split across ranks (NEXT-4: trials are
    independent counter-based streams, so rank r runs trials [t0, t0 + n) and
    the per-trial results equal a single-GPU run's).  Returns (t0, n)."""
    if not (0 <= rank < world) or trials < 0:
        raise ValueError("bad rank/world/trials")
    base, extra = divmod(trials, world)
    t0 = rank * base + min(rank, extra)
    return t0, base + (1 if rank < extra else 0)


def reduce_exceed(local):
    """Sum the per-plan exceedance counts (int64 tensor) over ranks: the one
    collective of a sharded Monte Carlo verification."""
    import torch.distributed as dist
    if dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(local, op=dist.ReduceOp.SUM)
    return local


def row_block(rank: int, world: int, n: int):
    """Rows [b, e) of rank `rank` in a row-sharded build of n rows."""
    if not (0 <= rank < world) or n < 0:
        raise ValueError("bad rank/world/n")
    base, extra = divmod(n, world)
    b = rank * base + min(rank, extra)
    return b, b + base + (1 if rank < extra else 0)


def csr_block(full: dict, b: int, e: int) -> dict:
    """The block of rows [b, e) of an exported CSR (row counts + the rows'
    edge arrays, dst | coll << 31 packed as in the C ABI)."""
    rp = np.asarray(full["row_ptr"], dtype=np.int64)
    lo, hi = int(rp[b]), int(rp[e])
    dc = (np.asarray(full["dst"][lo:hi], dtype=np.uint32) |
          (np.asarray(full["coll"][lo:hi], dtype=np.uint32) << np.uint32(31)))
    return {"b": b, "e": e, "counts": np.diff(rp[b:e + 1]).astype(np.int32), "dst_coll": dc,
            "w": np.asarray(full["w"][lo:hi], np.float32), "s": np.asarray(full["s"][lo:hi], np.float32),
            "c": np.asarray(full["c"][lo:hi], np.float32)}


def assemble_csr(blocks, n: int) -> dict:
    """Concatenate row blocks (any order; they must tile [0, n)) into one CSR:
    row_ptr [n+1] int32, dst_coll, w, s, c."""
    blocks = sorted(blocks, key=lambda k: k["b"])
    if blocks[0]["b"] != 0 or blocks[-1]["e"] != n or any(x["e"] != y["b"] for x, y in zip(blocks, blocks[1:])):
        raise ValueError("row blocks do not tile [0, n)")
    counts = np.concatenate([k["counts"] for k in blocks])
    row_ptr = np.zeros(n + 1, np.int64)
    np.cumsum(counts, out=row_ptr[1:])
    cat = {f: np.concatenate([k[f] for k in blocks]) for f in ("dst_coll", "w", "s", "c")}
    return {"row_ptr": row_ptr.astype(np.int32), **cat}


def gather_csr_blocks(block: dict, world: int):
    """All-gather every rank's CSR block (one collective round: sizes, then the
    padded 16-byte edge records and row counts)."""
    import torch
    import torch.distributed as dist
    if world == 1:
        return [block]
    dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend() == "nccl" else torch.device("cpu")
    meta = torch.tensor([block["b"], block["e"], block["dst_coll"].size], dtype=torch.int64, device=dev)
    metas = [torch.empty_like(meta) for _ in range(world)]
    dist.all_gather(metas, meta)
    metas = [m.cpu().numpy() for m in metas]
    max_rows = int(max(m[1] - m[0] for m in metas))
    max_nnz = int(max(m[2] for m in metas))
    rec = np.zeros((max(max_nnz, 1), 4), np.uint32)
    nnz = block["dst_coll"].size
    rec[:nnz, 0] = block["dst_coll"]
    for j, f in enumerate(("w", "s", "c")):
        rec[:nnz, j + 1] = block[f].view(np.uint32)
    cnt = np.zeros(max(max_rows, 1), np.int32)
    cnt[: block["counts"].size] = block["counts"]
    t_rec = torch.from_numpy(rec.view(np.int32)).to(dev)
    t_cnt = torch.from_numpy(cnt).to(dev)
    recs = [torch.empty_like(t_rec) for _ in range(world)]
    cnts = [torch.empty_like(t_cnt) for _ in range(world)]
    dist.all_gather(recs, t_rec)
    dist.all_gather(cnts, t_cnt)
    out = []
    for m, r_, c_ in zip(metas, recs, cnts):
        b, e, k = int(m[0]), int(m[1]), int(m[2])
        r_ = r_.cpu().numpy().view(np.uint32)[:k]
        out.append({"b": b, "e": e, "counts": c_.cpu().numpy()[: e - b], "dst_coll": r_[:, 0].copy(),
                    "w": r_[:, 1].copy().view(np.float32), "s": r_[:, 2].copy().view(np.float32),
                    "c": r_[:, 3].copy().view(np.float32)})
    return out


def gather_csr_blocks_device(part, b: int, e: int, world: int, n: int, positions, r: float, stream=None):
    """Device-resident row-sharded assembly: this rank's
    block of rows [b, e) of `part` (a mpap_build_roadmap_rows roadmap) is
    written into CUDA tensors (mpap_roadmap_block_device), all-gathered with
    two NCCL all_gather_into_tensor calls (row counts, 16-byte records; slots
    padded to the largest block, sizes agreed by one all-reduce MAX), and
    assembled on the device (mpap_roadmap_assemble_device).  Returns the
    search roadmap; the CSR never visits the host."""
    import torch
    import torch.distributed as dist
    from . import mpap_roadmap_assemble_device, mpap_roadmap_block_device, mpap_roadmap_info
    dev = torch.device("cuda", torch.cuda.current_device())
    nnz = mpap_roadmap_info(part)["nnz"]
    size = torch.tensor([e - b, nnz], dtype=torch.int64, device=dev)
    if world > 1:
        dist.all_reduce(size, op=dist.ReduceOp.MAX)
    rows_max, nnz_max = int(size[0].item()), max(int(size[1].item()), 1)
    counts = torch.zeros(rows_max, dtype=torch.int32, device=dev)
    edges = torch.zeros((nnz_max, 4), dtype=torch.int32, device=dev)
    mpap_roadmap_block_device(part, counts, edges, stream=stream)
    if world > 1:
        gc = torch.empty(world * rows_max, dtype=torch.int32, device=dev)
        ge = torch.empty((world * nnz_max, 4), dtype=torch.int32, device=dev)
        dist.all_gather_into_tensor(gc, counts)
        dist.all_gather_into_tensor(ge, edges)
    else:
        gc, ge = counts, edges
    row_begin = [row_block(g, world, n)[0] for g in range(world)] + [n]
    return mpap_roadmap_assemble_device(positions, row_begin, gc.view(world, rows_max),
                                        ge.view(world, nnz_max, 4), r, stream=stream)
