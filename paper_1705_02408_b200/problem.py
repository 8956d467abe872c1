"""Marshalling helpers: synth.Problem objects -> the C ABI calls.

Argument packing only (no arithmetic of the method); used by tests, smoke()
and bench.py.
"""
from __future__ import annotations

from typing import Any, Dict, List, Sequence

import numpy as np

from . import (MPAP_MEM_DEVICE, Roadmap, mpap_build_roadmap, mpap_build_roadmap_batch, mpap_build_roadmap_rows,
               mpap_mc_verify_batch, mpap_roadmap_export, mpap_roadmap_import,
               mpap_search, mpap_search_batch, params_from_problem)


def build_problem(prob, stream=None, edge_peaks: bool = False, lazy_edges: bool = False) -> Roadmap:
    prm, keep = params_from_problem(prob, edge_peaks, lazy_edges)
    obst = prob.obstacles if prob.obstacles.size else None
    feat = prob.features if prob.features.size else None
    rm = mpap_build_roadmap(prob.samples, obst if obst is not None else np.zeros((0, 2 * prob.pos_dim)),
                            feat if feat is not None else np.zeros((0, prob.pos_dim)), prob.r, prm, stream=stream)
    del keep
    return rm


def build_problem_rows(prob, row_begin: int, row_end: int, stream=None) -> Roadmap:
    """Row-sharded build of one environment (rows [row_begin, row_end))."""
    prm, keep = params_from_problem(prob)
    obst = prob.obstacles if prob.obstacles.size else np.zeros((0, 2 * prob.pos_dim))
    feat = prob.features if prob.features.size else np.zeros((0, prob.pos_dim))
    rm = mpap_build_roadmap_rows(prob.samples, obst, feat, prob.r, prm, row_begin, row_end, stream=stream)
    del keep
    return rm


def build_problem_sharded(prob, rank: int, world: int, stream=None) -> Roadmap:
    """rank builds its row block, the blocks are all-gathered
    (one collective) and concatenated, and every rank wraps the full CSR for
    search (mpap_roadmap_import: search-only, no geometry)."""
    from .dist import assemble_csr, csr_block, gather_csr_blocks, row_block
    b, e = row_block(rank, world, prob.n)
    part = build_problem_rows(prob, b, e, stream=stream)
    block = csr_block(mpap_roadmap_export(part), b, e)
    part.free()
    full = assemble_csr(gather_csr_blocks(block, world), prob.n)
    return mpap_roadmap_import(prob.samples[:, : prob.pos_dim], full["row_ptr"], full["dst_coll"], full["w"],
                               full["s"], full["c"], prob.r, stream=stream)


def build_problem_sharded_device(prob, rank: int, world: int, stream=None) -> Roadmap:
    """SURVEY.md §8(e) with the CSR blocks kept on the device: build rows
    [g n/G, (g+1) n/G), one NCCL all-gather of the device blocks, device-side
    assembly (dist.gather_csr_blocks_device)."""
    from .dist import gather_csr_blocks_device, row_block
    b, e = row_block(rank, world, prob.n)
    part = build_problem_rows(prob, b, e, stream=stream)
    try:
        return gather_csr_blocks_device(part, b, e, world, prob.n, prob.samples[:, : prob.pos_dim], prob.r,
                                        stream=stream)
    finally:
        part.free()


def search_problem(rm: Roadmap, prob, beta: float, env: int = 0, lam=None, trace_waves: int = 0,
                   path_capacity: int = 65536, stream=None, forall_t: bool = False) -> Dict[str, Any]:
    return mpap_search(rm, env, prob.start, prob.goal_lo, prob.goal_hi, beta, prob.lam if lam is None else lam,
                       path_capacity=path_capacity, trace_waves=trace_waves, stream=stream, forall_t=forall_t)


class Batch:
    """Concatenated host arrays of a list of problems sharing params and r."""

    def __init__(self, probs: Sequence[Any], edge_peaks: bool = False):
        p0 = probs[0]
        self.probs = list(probs)
        self.stride = p0.stride
        self.n = np.array([p.n for p in probs], np.int32)
        self.n_obst = np.array([p.obstacles.shape[0] for p in probs], np.int32)
        self.n_feat = np.array([p.features.shape[0] for p in probs], np.int32)
        self.samples = np.ascontiguousarray(np.concatenate([p.samples for p in probs]), np.float64)
        self.obstacles = np.ascontiguousarray(np.concatenate([p.obstacles.reshape(-1) for p in probs]), np.float64)
        self.features = np.ascontiguousarray(np.concatenate([p.features.reshape(-1) for p in probs]), np.float64)
        self.prm, self._keep = params_from_problem(p0, edge_peaks)
        self.r = p0.r
        self.lam = p0.lam
        self.starts = np.array([p.start for p in probs], np.int32)
        self.goals_lo = [p.goal_lo for p in probs]
        self.goals_hi = [p.goal_hi for p in probs]

    @property
    def h2d_bytes(self) -> int:
        return int(self.samples.nbytes + self.obstacles.nbytes + self.features.nbytes)

    def build(self, samples=None, obstacles=None, features=None, stream=None) -> Roadmap:
        """Host arrays by default; pass CUDA tensors for device-resident inputs."""
        return mpap_build_roadmap_batch(self.samples if samples is None else samples, self.n, self.stride,
                                        self.obstacles if obstacles is None else obstacles, self.n_obst,
                                        self.features if features is None else features, self.n_feat, self.r,
                                        self.prm, stream=stream)

    def search(self, rm: Roadmap, betas: Sequence[float], path_capacity: int = 1024, paths=None, results=None,
               stream=None, envs=None, trace_waves: int = 0):
        """One query per environment (envs=None) or the given environment
        index per query; betas per query."""
        envs = np.arange(len(self.probs), dtype=np.int32) if envs is None else np.asarray(envs, np.int32)
        return mpap_search_batch(rm, envs, self.starts[envs], [self.goals_lo[e] for e in envs],
                                 [self.goals_hi[e] for e in envs], betas, self.lam, path_capacity, paths=paths,
                                 results=results, stream=stream, trace_waves=trace_waves)

    def mc_verify(self, rm: Roadmap, paths, results, mc: Dict[str, Any], trial0: int = 0, per_trial: bool = False,
                  stream=None):
        """Monte Carlo verification (NEXT-4) of every feasible plan of a
        search batch (host paths/results as returned by ``search``); returns
        (env indices, MC results, per-trial max errors or None)."""
        ok = np.nonzero(results["status"] == 0)[0].astype(np.int32)
        if ok.size == 0:
            return ok, None, None
        res, me, _ = mpap_mc_verify_batch(rm, ok, paths[ok], results["path_len"][ok], mc, trial0=trial0,
                                          per_trial=per_trial, stream=stream)
        return ok, res, me


# ---------------------------------------------------------------------------
# NEXT-2: batched perception-bound sweep and refinement.
# Alg. 1 line 4 re-runs Explore with an updated beta; with one
# roadmap resident, many betas run as one batched launch (one CTA per beta).
# ---------------------------------------------------------------------------

def beta_sweep(rm: Roadmap, prob, betas: Sequence[float], env: int = 0, path_capacity: int = 1024,
               stream=None, forall_t: bool = False):
    """Explore (Alg. 3) for every beta in one batched launch on one roadmap;
    returns (paths [len(betas), cap], result records)."""
    nb = len(betas)
    envs = np.full(nb, env, dtype=np.int32)
    starts = np.full(nb, prob.start, dtype=np.int32)
    return mpap_search_batch(rm, envs, starts, [prob.goal_lo] * nb, [prob.goal_hi] * nb,
                             np.asarray(betas, dtype=np.float64), prob.lam, path_capacity, stream=stream,
                             forall_t=forall_t)


def refine_beta_min(rm: Roadmap, prob, hi: float, rel_tol: float = 1e-3, per_round: int = 32, env: int = 0,
                    max_rounds: int = 20):
    """Smallest perception bound with a feasible plan, to `rel_tol` relative:
    each round evaluates `per_round` equally spaced bounds in [lo, hi] with one
    batched launch and keeps the bracket around the feasibility switch
    (Explore feasibility is monotone in beta).  Returns (lo, hi, rounds):
    infeasible at lo (or lo == 0), feasible at hi."""
    _, r = beta_sweep(rm, prob, [hi], env)
    if r[0]["status"] != 0:
        raise ValueError("no feasible plan even at the upper bound")
    _, r0 = beta_sweep(rm, prob, [0.0], env)
    if r0[0]["status"] == 0:
        return 0.0, 0.0, 1
    lo = 0.0
    rounds = 0
    while hi - lo > rel_tol * hi and rounds < max_rounds:
        grid = lo + (hi - lo) * np.arange(1, per_round + 1) / (per_round + 1)
        _, res = beta_sweep(rm, prob, grid, env)
        feas = res["status"] == 0
        k = int(np.argmax(feas)) if feas.any() else per_round
        new_hi = grid[k] if k < per_round else hi
        new_lo = grid[k - 1] if k > 0 else lo
        lo, hi = float(new_lo), float(new_hi)
        rounds += 1
    return lo, hi, rounds


# ---------------------------------------------------------------------------
# NEXT-2 + NEXT-4: Alg. 1 line 4, "MC sampling and refinement of bound for
# Alg. 3" ("the perception-heuristic bound may be updated ... and
# the exploration rerun").  A grid of bounds runs as one batched search; the
# distinct feasible plans run as one batched Monte Carlo launch; the certified
# plan is the one of the largest bound whose plan passes p_hat <= alpha
# (lowest cost among certified plans: Explore's cost is non-increasing in beta
# up to its group approximation, so the largest passing bound is selected
# explicitly rather than by bisection).
# ---------------------------------------------------------------------------

def refine_beta_mc(rm: Roadmap, prob, betas: Sequence[float], mc: Dict[str, Any], alpha: float, env: int = 0,
                   path_capacity: int = 1024, stream=None) -> Dict[str, Any]:
    betas = np.sort(np.asarray(betas, dtype=np.float64))
    paths, res = beta_sweep(rm, prob, betas, env, path_capacity=path_capacity, stream=stream)
    plans: Dict[tuple, int] = {}
    for k in range(len(betas)):
        if res["status"][k] == 0:
            plans.setdefault(tuple(paths[k][: res["path_len"][k]].tolist()), len(plans))
    table = []
    best = None
    if plans:
        keys = list(plans.keys())
        cap = max(len(p) for p in keys)
        pa = np.zeros((len(keys), cap), dtype=np.int32)
        for i, p in enumerate(keys):
            pa[i, : len(p)] = p
        mres, _, _ = mpap_mc_verify_batch(rm, np.full(len(keys), env, np.int32), pa, [len(p) for p in keys], mc,
                                          per_trial=False, stream=stream)
        for k in range(len(betas)):
            row = {"beta": float(betas[k]), "status": int(res["status"][k])}
            if res["status"][k] == 0:
                i = plans[tuple(paths[k][: res["path_len"][k]].tolist())]
                row.update(cost=float(res["cost"][k]), h=float(res["h"][k]), p_hat=float(mres["p_hat"][i]),
                           plan=i, passed=bool(mres["p_hat"][i] <= alpha))
                if row["passed"]:
                    best = k
            table.append(row)
    else:
        table = [{"beta": float(b), "status": int(s)} for b, s in zip(betas, res["status"])]
    out = {"table": table, "certified": best is not None}
    if best is not None:
        out.update(beta=float(betas[best]), path=paths[best][: res["path_len"][best]].copy(),
                   cost=float(res["cost"][best]), p_hat=table[best]["p_hat"])
    return out
