#!/usr/bin/env python
"""bench.py -- MPAP hot path on B200: batched roadmap build + search.

Metric (BASELINE.json): "edges relaxed/sec and queries/sec at 1/2/4/8 B200;
HBM roofline fraction".  Workload: C5 (BASELINE.json configs[4]), the 6D
double-integrator quadrotor named by north_star, weak-scaled: each rank
processes its own shard of `queries_per_gpu` independent environment+query
units (env seeds 1000 + rank*Q + k), so 8 GPUs x 64 = C5's 512 queries.

One step = one pass of the whole hot path over
the rank's batch: mpap_build_roadmap_batch (neighbours, collision, heuristic,
CSR) + mpap_search_batch (Alg. 3 for every query) + the NCCL all-gather of the
fixed-size result records (N > 1; the only collective, never inside the wave
loop).  `value` = queries of all ranks / max-over-ranks device time, inputs
resident in HBM; `e2e` = the same through the C ABI with pinned HOST buffers
(H2D of the inputs and D2H of the results inside the timed region).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl mpap|reference]
                    [--queries-per-gpu Q] [--rowshard] [--launcher-selftest]

--gpus N (N > 1) outside torchrun re-launches this script as N ranks under
torch.distributed.run (one process per GPU, NCCL, 127.0.0.1 rendezvous);
rank 0 prints the one JSON line.  Every run ends with a hard parity gate:
the timed step's results (and, outside the timed region, the same batch's
per-wave counters and CSR digests) are compared with the oracle's stored
outputs (tests/golden/, written by tests/golden/make_golden.py, oracle only)
or, for environments no golden covers, with the oracle run live; a mismatch
prints the line with "parity_gate": {"passed": false, ...} and exits 3.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = json.load(open(os.path.join(ROOT, "BASELINE.json")))["metric"]
PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
FALLBACK_HBM_GBS = 6650.0
# FP64 issue peak for a non-FMA DADD/DMUL stream: 148 SMs x 64 FP64 lanes x clock
# (B200: FP64 = half the FP32 lane count; DESIGN.md §7 derivation).
SMS = 148
FP64_LANES_PER_SM = 64


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="mpap", choices=["mpap", "reference"])
    ap.add_argument("--config", default="c5")
    ap.add_argument("--queries-per-gpu", type=int, default=0)
    ap.add_argument("--beta", type=float, default=float("nan"))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-procs", type=int, default=0)
    ap.add_argument("--no-mc", action="store_true", help="skip the Monte Carlo verification measurement")
    ap.add_argument("--no-lazy", action="store_true", help="skip the lazy-roadmap variant measurement")
    ap.add_argument("--mc-trials", type=int, default=1000)
    ap.add_argument("--rowshard", action="store_true",
                    help="time the row-sharded build of one large roadmap (default config c4) instead")
    ap.add_argument("--launcher-selftest", action="store_true",
                    help="CPU/gloo check of the rank launcher and the result gather (no GPU work)")
    ap.add_argument("--no-gate", action="store_true", help="diagnostics only: skip the parity gate")
    return ap.parse_args()


# ---------------------------------------------------------------------------
# rank launcher: --gpus N outside torchrun -> N processes under torchrun
# ---------------------------------------------------------------------------
def spawn_ranks(n: int) -> int:
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")          # stderr: shows the NVLink/NVLS transport NCCL picked
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    env.setdefault("OMP_NUM_THREADS", "1")
    return subprocess.call(cmd, env=env)


def launcher_selftest(args) -> int:
    """Ranks started by spawn_ranks (or torchrun) on CPU with gloo: every rank
    writes its shard's fixed-size result records, the records are gathered with
    the bench's collective (dist.gather_results) and the step time is reduced
    MAX over ranks, exactly as in the GPU bench; rank 0 prints one line."""
    import torch
    import torch.distributed as dist
    from paper_1705_02408_b200.dist import shard_envs
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world > 1:
        dist.init_process_group("gloo")
    Q = args.queries_per_gpu or 4
    envs = shard_envs(rank, world, Q)
    rec = np.zeros(Q, dtype=np.dtype([("env", np.int64), ("rank", np.int64), ("pad", np.int64, 4)]))
    rec["env"] = envs
    rec["rank"] = rank
    local = torch.from_numpy(rec.view(np.uint8).copy())
    if world > 1:
        from paper_1705_02408_b200.dist import gather_results
        allrec = gather_results(local, world).numpy().view(rec.dtype)
        t = torch.tensor([1.0 + rank], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t_max = float(t.item())
    else:
        allrec, t_max = rec, 1.0
    ok = allrec["env"].tolist() == list(range(world * Q)) and allrec["rank"].tolist() == \
        [r for r in range(world) for _ in range(Q)]
    if rank == 0:
        print(json.dumps({"launcher_selftest": True, "n_gpus": world, "gathered_queries": int(allrec.size),
                          "records_in_rank_order": bool(ok), "max_over_ranks": t_max}), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0 if ok else 3


# ---------------------------------------------------------------------------
# clocks during the timed region (B200_PROFILING.md clocks line)
# ---------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.path = None

    def start(self):
        if self.idx < 0:       # disabled (diagnostic runs only)
            return
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.idx}", f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        out = {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        if self.proc is None:
            return out
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax.append(float(parts[2]))
            except ValueError:
                continue
            for k, nm in enumerate(names):
                if parts[5 + k].lower().startswith("active"):
                    reasons.add(nm)
        os.unlink(self.path)
        if sm:
            out = {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(smax), "reasons": sorted(reasons),
                   "samples": len(sm)}
        return out


def load_peaks():
    try:
        pk = json.load(open(PEAKS_PATH))
        return pk, "measured"
    except Exception:
        return {"hbm_gbs": FALLBACK_HBM_GBS, "sm_max_mhz": 1965.0}, "fallback"


# ---------------------------------------------------------------------------
# workload
# ---------------------------------------------------------------------------
def make_shard(cfg, rank: int, world: int, Q: int):
    from paper_1705_02408_b200.dist import shard_envs
    from synth import make_problem
    return [make_problem(cfg, env_index=e) for e in shard_envs(rank, world, Q)]


def cpu_baseline(cfg, beta: float, procs: int, gpu_env0=None, gpu_path0=None):
    """The oracle as it stands on one environment+query of the workload:
    build rows spread over `procs` processes (each the sequential oracle),
    search single-threaded.  With the GPU's result record and plan for env 0
    of the timed step, also reports the parity gate (status, plan, cost and
    perception bits, relaxations equal)."""
    import oracle
    from synth import make_problem
    oracle.build()
    prob = make_problem(cfg, env_index=0)
    t0 = time.perf_counter()
    rm = oracle.build_roadmap_parallel(prob, procs)
    t1 = time.perf_counter()
    res = oracle.search(rm, prob, beta)
    t2 = time.perf_counter()
    out = {"value": 1.0 / (t2 - t0), "unit": "queries/s", "cores": procs, "kind": "oracle",
           "sample": f"1 {cfg['name']} environment+query (env 0, n={prob.n}): oracle build {t1 - t0:.2f} s "
                     f"over {procs} processes + oracle search {t2 - t1:.3f} s (1 thread), beta={beta}",
           "edges_relaxed_per_s": res["relaxations"] / (t2 - t0),
           "search_only_edges_relaxed_per_s": res["relaxations"] / max(t2 - t1, 1e-9)}
    if gpu_env0 is not None:
        g = gpu_env0
        ok = int(g["status"]) == int(res["status"]) and int(g["relaxations"]) == int(res["relaxations"])
        if ok and res["status"] == 0:
            ok = (gpu_path0.tolist() == res["path"].tolist()
                  and np.float32(g["cost"]).view(np.uint32) == np.float32(res["cost"]).view(np.uint32)
                  and np.float32(g["h"]).view(np.uint32) == np.float32(res["h"]).view(np.uint32))
        out["parity_gate_env0"] = bool(ok)
    return out


def run_reference(args, cfg, beta):
    """--impl reference: the oracle (CPU) timed as the reference arm."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    procs = args.cpu_procs or os.cpu_count() or 1
    import oracle
    from synth import make_problem
    oracle.build()
    prob = make_problem(cfg, env_index=0)
    times = []
    relax = 0
    for it in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        rm = oracle.build_roadmap_parallel(prob, procs)
        res = oracle.search(rm, prob, beta)
        dt = time.perf_counter() - t0
        if it >= args.warmup:
            times.append(dt)
            relax += res["relaxations"]
    tot = sum(times)
    value = args.steps / tot
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "queries/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64+f32",
        "data": "synthetic",
        "config": {"workload": f"{cfg['name']}: 1 environment+query per step (bounded sample of the GPU arm's "
                               f"workload), n={prob.n}", "beta": beta, "lambda": cfg.get("lambda", 0.5)},
        "edges_relaxed_per_s": relax / tot,
        "cpu_baseline": {"value": value, "unit": "queries/s", "cores": procs, "kind": "oracle",
                         "sample": f"1 {cfg['name']} environment+query per step: oracle build over {procs} "
                                   f"processes + oracle search (1 thread)"},
        "e2e": {"value": value, "unit": "queries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def main():
    args = parse()
    if args.impl == "mpap" and args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn_ranks(args.gpus)
    if args.launcher_selftest:
        return launcher_selftest(args)
    from synth import load_config
    if args.rowshard and args.config == "c5":
        args.config = "c4"
    cfg = load_config(args.config)
    beta = args.beta if not math.isnan(args.beta) else float(cfg["betas"][1])
    if args.impl == "reference":
        return run_reference(args, cfg, beta)
    if args.rowshard:
        return run_rowshard(args, cfg, beta)

    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    import build_ext
    if rank == 0 or world == 1:
        build_ext.build()
    if world > 1:
        dist.barrier()
    import paper_1705_02408_b200 as mp
    from paper_1705_02408_b200.dist import gather_results
    from paper_1705_02408_b200.problem import Batch

    Q = args.queries_per_gpu or int(cfg.get("queries_per_gpu", 64))
    probs = make_shard(cfg, rank, world, Q)
    B = Batch(probs)
    betas = [beta] * Q
    PATH_CAP = 512
    s_d = torch.from_numpy(B.samples).to(dev)
    o_d = torch.from_numpy(B.obstacles).to(dev)
    f_d = torch.from_numpy(B.features).to(dev)
    paths_d = torch.zeros((Q, PATH_CAP), dtype=torch.int32, device=dev)
    res_d = torch.zeros(Q * 48, dtype=torch.uint8, device=dev)
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream()

    last_work = {}

    def step_device():
        rm = B.build(s_d, o_d, f_d)
        B.search(rm, betas, path_capacity=PATH_CAP, paths=paths_d, results=res_d)
        if world > 1:
            gather_results(res_d, world)
        last_work.update(mp.mpap_roadmap_work(rm))
        rm.free()

    for _ in range(args.warmup):
        step_device()
    torch.cuda.synchronize()

    # ---- timed region: device-resident inputs ----
    sampler = ClockSampler(local) if os.environ.get("MPAP_BENCH_CLOCKS", "1") != "0" else ClockSampler(-1)
    mp.mpap_prof_reset()
    mp.mpap_prof_enable(True)
    launches0 = mp.mpap_launch_count()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    sampler.start()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    wall0 = time.perf_counter()
    host_ms = []
    for k in range(args.steps):
        flush.zero_()                      # L2 flush (512 MiB > 126 MB L2), outside the step's events
        ev[k][0].record(stream)
        h0 = time.perf_counter()
        step_device()
        host_ms.append((time.perf_counter() - h0) * 1e3)
        ev[k][1].record(stream)
    torch.cuda.synchronize()
    wall = time.perf_counter() - wall0
    if world > 1:
        dist.barrier()
    clocks = sampler.stop()
    mp.mpap_prof_enable(False)
    launches = mp.mpap_launch_count() - launches0
    step_ms = [a.elapsed_time(b) for a, b in ev]
    tot_ms = float(sum(step_ms))
    kern = {k: mp.mpap_prof_read(k) for k in mp.KERNELS}

    # results of the last step (outside the timed region)
    res = res_d.cpu().numpy().view(mp.RESULT_DTYPE)
    paths_h = paths_d.cpu().numpy()
    relax_step = int(res["relaxations"].sum())
    feasible = int((res["status"] == 0).sum())
    ok = bool(np.all((res["status"] == 0) | (res["status"] == 3)))

    t_max = torch.tensor([tot_ms], dtype=torch.float64, device=dev)
    r_sum = torch.tensor([relax_step, feasible], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t_max, op=dist.ReduceOp.MAX)
        dist.all_reduce(r_sum, op=dist.ReduceOp.SUM)
    tot_ms_max = float(t_max.item())
    relax_all = float(r_sum[0].item())
    feasible_all = int(r_sum[1].item())
    total_queries = world * Q * args.steps
    value = total_queries / (tot_ms_max / 1e3)
    search_ms = kern["k_search"][0]

    # ---- e2e: pinned HOST buffers through the C ABI ----
    e2e = None
    if not args.no_e2e:
        s_h = torch.from_numpy(B.samples).pin_memory()
        o_h = torch.from_numpy(B.obstacles).pin_memory()
        f_h = torch.from_numpy(B.features).pin_memory()
        h2d = int(s_h.numel() * 8 + o_h.numel() * 8 + f_h.numel() * 8 + Q * (4 * 2 + 8 + 48))
        d2h = int(Q * (48 + 4 * PATH_CAP))

        def step_host():
            rm = B.build(s_h, o_h, f_h)
            B.search(rm, betas, path_capacity=PATH_CAP)
            rm.free()

        step_host()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e_ms = 0.0
        for _ in range(args.steps):
            flush.zero_()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            step_host()
            b.record(stream)
            b.synchronize()
            e_ms += a.elapsed_time(b)
        te = torch.tensor([e_ms], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e = {"value": world * Q * args.steps / (float(te.item()) / 1e3), "unit": "queries/s",
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h}

    # ---- roofline of the dominant kernel ----
    peaks, peak_src = load_peaks()
    fp64 = measure_fp64_peak(mp)
    dom = max(mp.KERNELS, key=lambda k: kern[k][0])
    dom_ms, dom_n = kern[dom]
    roof = roofline(dom, dom_ms, dom_n, last_work, B, res, peaks, peak_src, fp64)
    roof["share_of_step"] = dom_ms / tot_ms if tot_ms > 0 else None
    if dom == "k_heuristic" and last_work:
        # context: SURVEY 8(d) writes the heuristic's work as K x F (step, feature)
        # pairs per edge; the exact chunk culls leave the executed
        # range tests -- the counted work above counts only executed tests
        pairs = float(last_work["steps"]) * float(np.mean(B.n_feat))
        roof["cull"] = {"step_feature_pairs_in_definition": pairs,
                        "range_tests_executed": int(last_work["range_tests"]),
                        "skipped_fraction": 1.0 - float(last_work["range_tests"]) / pairs if pairs else None}
    roof["traffic"] = committed_traffic(dom, Q)

    # ---- parity gate (hard): timed results, per-wave counters, CSR digests ----
    gate = {"passed": True, "skipped": True}
    gold = golden_index(cfg, beta)
    if not args.no_gate:
        gate = parity_gate(mp, B, probs, rank, world, Q, cfg, beta, gold, res, paths_h, s_d, o_d, f_d, PATH_CAP,
                           args)
        g = torch.tensor([1.0 if gate["passed"] else 0.0], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(g, op=dist.ReduceOp.MIN)
        gate["passed_all_ranks"] = bool(g.item() == 1.0)

    # the metric's "HBM roofline fraction" for the search itself (k_search):
    # SURVEY §8(d) algorithmic bytes 16 E_rows + 12 sum G + 8 F_reads + 16 L_ins
    # (oracle counters, stored with the goldens), and the simpler 16 B per
    # relaxation + 16 B per inserted label beside it
    search_roof = roofline("k_search", kern["k_search"][0], kern["k_search"][1], last_work, B, res, peaks, peak_src,
                           fp64, alg_bytes=search_alg_bytes(gold, rank, Q))
    search_roof["traffic"] = committed_traffic("k_search", Q)

    line = {
        "metric": METRIC, "value": value, "unit": "queries/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": tot_ms_max / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64+f32", "data": "synthetic",
        "config": {"workload": f"{cfg['name']} shard: {Q} independent 6D double-integrator quadrotor "
                               f"environments+queries per GPU (n={B.n.max()}, {int(B.n_obst.max())} boxes, "
                               f"{int(B.n_feat.max())} features, MLP heuristic); build+search per step",
                   "queries_per_gpu": Q, "global_queries_per_step": world * Q, "beta": beta,
                   "lambda": B.lam, "r": B.r, "parallelism": f"dp{world} (independent queries)",
                   "l2": "flushed between timed steps (512 MiB write, outside the step events)"},
        "edges_relaxed_per_s": relax_all * args.steps / (tot_ms_max / 1e3),
        "search_only": {"roofline": search_roof,
                        "ms_per_step": search_ms / max(kern['k_search'][1], 1),
                        "edges_relaxed_per_s": relax_step / (search_ms / max(kern['k_search'][1], 1) / 1e3)
                        if search_ms > 0 else None,
                        "queries_per_s": Q / (search_ms / max(kern['k_search'][1], 1) / 1e3) if search_ms else None},
        "kernels_ms_per_step": {k: kern[k][0] / args.steps for k in mp.KERNELS},
        "feasible_fraction": feasible_all / (world * Q), "all_status_ok": ok,
        "roofline": roof, "fp64_peak_measured": fp64, "gpu_launches": int(launches), "clocks": clocks,
        "wall_s": wall, "step_ms": [round(x, 3) for x in step_ms],
        "step_ms_stats": step_stats(step_ms),
        "step_host_ms": [round(x, 3) for x in host_ms],
        "search_teams": mp.mpap_search_launches(),
        "parity_gate": gate,
    }
    if e2e:
        line["e2e"] = e2e
    if not args.no_lazy:
        line["lazy_variant"] = measure_lazy(mp, B, s_d, o_d, f_d, betas, PATH_CAP, paths_d, res_d, flush, args.steps,
                                            res, world)
    if not args.no_mc:
        line["mc_verify"] = measure_mc(mp, B, betas, PATH_CAP, args.mc_trials, rank == 0 and world == 1
                                       and not args.no_cpu_baseline)
    if (rank == 0) and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(cfg, beta, args.cpu_procs or os.cpu_count() or 1, res[0],
                                            paths_h[0][: int(res[0]["path_len"])])
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0 if gate.get("passed_all_ranks", gate["passed"]) else 3


# ---------------------------------------------------------------------------
# parity gate
# ---------------------------------------------------------------------------
GOLDEN_DIR = os.path.join(ROOT, "tests", "golden")


def golden_index(cfg, beta):
    """{global env index: oracle record of the search at `beta`} from the
    stored goldens (c5_bench.json: envs 0..63 at four bounds; c5_all.json:
    every C5 environment at the bench bound), plus the environments' CSR
    digests.  Empty for other configs or bounds."""
    out = {}
    if cfg["name"] != "c5":
        return out
    for fn in ("c5_all.json", "c5_bench.json"):
        path = os.path.join(GOLDEN_DIR, fn)
        if not os.path.exists(path):
            continue
        g = json.load(open(path))
        for env in g["envs"]:
            k = int(env["name"].split("[")[1].rstrip("]"))
            for srch in env["searches"]:
                b = float("inf") if srch["beta"] == "inf" else float(srch["beta"])
                if b == beta:
                    out[k] = {"search": srch, "digests": env.get("digests"), "nnz": env["nnz"]}
    return out


def _f32hex(x):
    return np.float32(x).tobytes().hex()


def _same(rec, path, s, counters=None):
    if int(rec["status"]) != s["status"] or int(rec["waves"]) != s["waves"]:
        return False
    if int(rec["relaxations"]) != s["relaxations"] or int(rec["labels_inserted"]) != s["labels_inserted"]:
        return False
    if s["status"] == 0:
        if path.tolist() != s["path"] or _f32hex(rec["cost"]) != s["cost"] or _f32hex(rec["h"]) != s["h"]:
            return False
        if _f32hex(rec["h_peak"]) != s["h_peak"]:
            return False
    if counters is not None and counters.tolist() != s["wave_counters"]:
        return False
    return True


def parity_gate(mp, B, probs, rank, world, Q, cfg, beta, gold, res, paths_h, s_d, o_d, f_d, path_cap, args):
    """Bit-exact comparison of this rank's timed-step results with the oracle
    (SURVEY §8(d) "parity gates in every benchmark run"): every environment of
    the shard a golden covers (status, waves, relaxations, inserted labels,
    plan, cost / h / h_peak bits); outside the timed region the same batch is
    rebuilt and searched once more with per-wave counters in the same launch
    configuration (mpap_search_batch_trace) and the CSR digests of up to 8
    covered environments are checked.  A shard no golden covers is checked
    against the oracle run live on its first environment."""
    sys.path.insert(0, GOLDEN_DIR)
    from digest import csr_digests
    envs = [rank * Q + k for k in range(Q)]
    covered = [k for k in range(Q) if envs[k] in gold]
    out = {"passed": True, "source": "golden" if covered else "oracle (live)", "envs_checked": 0,
           "wave_counters_checked": 0, "digests_checked": 0, "mismatches": []}
    rm = B.build(s_d, o_d, f_d)
    try:
        _, tres, tw = B.search(rm, [beta] * Q, path_capacity=path_cap, trace_waves=512)
        if covered:
            for k in covered:
                s = gold[envs[k]]["search"]
                pl = int(res[k]["path_len"]) if res[k]["status"] == 0 else 0
                if not _same(res[k], paths_h[k][:pl], s):
                    out["mismatches"].append(f"env {envs[k]}: timed result")
                if not _same(tres[k], paths_h[k][:pl], s, counters=tw[k]):
                    out["mismatches"].append(f"env {envs[k]}: traced result / wave counters")
                out["envs_checked"] += 1
                out["wave_counters_checked"] += 1
            for k in covered[:: max(1, len(covered) // 8)][:8]:
                if csr_digests(mp.mpap_roadmap_export(rm, k)) != gold[envs[k]]["digests"]:
                    out["mismatches"].append(f"env {envs[k]}: CSR digest")
                out["digests_checked"] += 1
        else:
            import oracle
            oracle.build()
            procs = max(1, (args.cpu_procs or os.cpu_count() or 1) // max(world, 1))
            orm = oracle.build_roadmap_parallel(probs[0], procs)
            o = oracle.search(orm, probs[0], beta)
            s = {"status": o["status"], "waves": o["waves"], "relaxations": o["relaxations"],
                 "labels_inserted": o["labels_inserted"], "path": o["path"].tolist(), "cost": _f32hex(o["cost"]),
                 "h": _f32hex(o["h"]), "h_peak": _f32hex(o["h_peak"]), "wave_counters": o["wave_counters"].tolist()}
            pl = int(res[0]["path_len"]) if res[0]["status"] == 0 else 0
            if not _same(res[0], paths_h[0][:pl], s) or not _same(tres[0], paths_h[0][:pl], s, counters=tw[0]):
                out["mismatches"].append(f"env {envs[0]}: result vs live oracle")
            g = mp.mpap_roadmap_export(rm, 0)
            if csr_digests(g) != csr_digests(orm):
                out["mismatches"].append(f"env {envs[0]}: CSR vs live oracle")
            out.update(envs_checked=1, wave_counters_checked=1, digests_checked=1)
    finally:
        rm.free()
    out["passed"] = not out["mismatches"]
    out["mismatches"] = out["mismatches"][:10]
    return out


def search_alg_bytes(gold, rank, Q):
    """SURVEY §8(d) algorithmic bytes of this rank's timed search, summed
    over its queries from the oracle's counters: 16 E_rows + 12 sum_i |G_i| +
    8 F_reads (clean staircase entries read) + 16 L_ins.  None unless every
    query of the shard has a golden record carrying E_rows."""
    tot = {"e_rows": 0, "sum_g": 0, "f_reads": 0, "l_ins": 0}
    for k in range(Q):
        g = gold.get(rank * Q + k)
        if g is None or "e_rows" not in g["search"]:
            return None
        s = g["search"]
        wc = np.asarray(s["wave_counters"], dtype=np.int64).reshape(-1, 8)
        tot["e_rows"] += int(s["e_rows"])
        tot["sum_g"] += int(wc[:, 1].sum())
        tot["f_reads"] += int(wc[:, 7].sum())
        tot["l_ins"] += int(s["labels_inserted"])
    tot["bytes"] = 16 * tot["e_rows"] + 12 * tot["sum_g"] + 8 * tot["f_reads"] + 16 * tot["l_ins"]
    return tot


def measure_fp64_peak(mp):
    """FP64 issue peak measured on this GPU (mpap_prof_fp64_peak: DFMA, DADD
    streams; one instruction = one counted op), in T ops/s."""
    out = {}
    for kind in ("dfma", "dadd"):
        ops, ms = mp.mpap_prof_fp64_peak(kind)
        out[kind + "_tops"] = ops / 1e12
    out["tops"] = max(out["dfma_tops"], out["dadd_tops"])
    return out


def run_rowshard(args, cfg, beta):
    """SURVEY §8(e) row-sharded precompute of ONE large roadmap (C4, n =
    16 001): rank g builds rows [g n/G, (g+1) n/G) (mpap_build_roadmap_rows),
    the CSR blocks are all-gathered once (dist.gather_csr_blocks) and
    concatenated in row order, every rank wraps the full CSR
    (mpap_roadmap_import) and runs the query.  Step = build block + gather +
    assemble + import + search; value = queries/s of the whole job (max over
    ranks).  Gate: the assembled CSR's digests and the search equal the
    oracle's stored C4 outputs."""
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    import build_ext
    if rank == 0 or world == 1:
        build_ext.build()
    if world > 1:
        dist.barrier()
    import paper_1705_02408_b200 as mp
    from paper_1705_02408_b200.dist import gather_csr_blocks_device, row_block
    from paper_1705_02408_b200.problem import build_problem_rows, search_problem
    from synth import make_problem
    prob = make_problem(cfg)
    b, e = row_block(rank, world, prob.n)
    stream = torch.cuda.current_stream()
    phases = {"build_block": 0.0, "gather_assemble_import": 0.0, "search": 0.0}
    state = {}

    def step(timed, keep=False):
        a = torch.cuda.Event(enable_timing=True)
        m = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        part = build_problem_rows(prob, b, e)
        m.record(stream)
        m.synchronize()
        t1 = time.perf_counter()
        # device-resident blocks: one NCCL all-gather, assembly on the device
        rm = gather_csr_blocks_device(part, b, e, world, prob.n, prob.samples[:, : prob.pos_dim], prob.r)
        part.free()
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        res = search_problem(rm, prob, beta, path_capacity=4096)
        t3 = time.perf_counter()
        if timed:
            phases["build_block"] += a.elapsed_time(m)
            phases["gather_assemble_import"] += (t2 - t1) * 1e3
            phases["search"] += (t3 - t2) * 1e3
        state["res"] = res
        if keep:
            state["full"] = mp.mpap_roadmap_export(rm)
        rm.free()

    for _ in range(args.warmup):
        step(False)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step(True)
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t0) * 1e3
    step(False, keep=True)   # the gate's copy of the assembled CSR, outside the timed steps
    t = torch.tensor([ms] + [phases[k] for k in phases], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t[0].item())
    # gate vs the oracle's stored C4 roadmap and search
    sys.path.insert(0, GOLDEN_DIR)
    from digest import csr_digests
    full, res = state["full"], state["res"]
    gate = {"passed": True, "skipped": True}
    gpath = os.path.join(GOLDEN_DIR, f"{cfg['name']}_full.json")
    if os.path.exists(gpath):
        gold = json.load(open(gpath))
        dig = csr_digests(full)
        srch = [x for x in gold["searches"] if x["beta"] != "inf" and float(x["beta"]) == beta]
        ok = dig == gold.get("digests")
        if srch:
            x = srch[0]
            ok = ok and res["status"] == x["status"] and res["relaxations"] == x["relaxations"] and \
                (x["status"] != 0 or (res["path"].tolist() == x["path"] and _f32hex(res["cost"]) == x["cost"]
                                      and _f32hex(res["h"]) == x["h"]))
        gate = {"passed": bool(ok), "digests_equal": dig == gold.get("digests"), "search_checked": bool(srch)}
    nnz = int(np.asarray(full["row_ptr"])[-1])
    if rank == 0:
        line = {"metric": METRIC + " (row-sharded single-roadmap build variant)", "value": args.steps / (ms_max / 1e3),
                "unit": "queries/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": ms_max / args.steps, "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "f64+f32", "data": "synthetic",
                "config": {"workload": f"{cfg['name']}: one roadmap n={prob.n} row-sharded over {world} GPU(s), one "
                                       f"device-resident CSR all-gather (NCCL) + device assembly, then the "
                                       f"single query at beta={beta}",
                           "rows_per_rank": e - b, "nnz": nnz},
                "phases_ms_per_step_max_over_ranks": {k: float(t[i + 1].item()) / args.steps
                                                      for i, k in enumerate(phases)},
                "edges_built_per_s": nnz * args.steps / (ms_max / 1e3),
                "parity_gate": gate}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0 if gate["passed"] else 3


def measure_lazy(mp, B, s_d, o_d, f_d, betas, path_cap, paths_d, res_d, flush, steps, res_eager, world=1):
    """NEXT-1 part i variant of the same step: the roadmap is built lazily
    (Near + Cost) and the batched search evaluates the rows its waves need
    (suspend / evaluate the union of requested rows / resume).  Same plans --
    checked record for record against the eager step's results; timed like the
    headline (CUDA events, L2 flushed, inputs resident), reported beside it,
    not as the headline."""
    import torch
    stream = torch.cuda.current_stream()
    rows = [0]

    def step():
        B.prm.lazy_edges = 1
        rm = B.build(s_d, o_d, f_d)
        B.prm.lazy_edges = 0
        B.search(rm, betas, path_capacity=path_cap, paths=paths_d, results=res_d)
        rows[0] = sum(mp.mpap_roadmap_rows_evaluated(rm, e) for e in range(len(B.probs)))
        rm.free()

    step()
    torch.cuda.synchronize()
    ms = 0.0
    mp.mpap_prof_reset()
    mp.mpap_prof_enable(True)
    l0 = mp.mpap_launch_count()
    for _ in range(steps):
        flush.zero_()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        step()
        b.record(stream)
        b.synchronize()
        ms += a.elapsed_time(b)
    mp.mpap_prof_enable(False)
    launches = mp.mpap_launch_count() - l0
    kern = {k: mp.mpap_prof_read(k) for k in mp.KERNELS + ("k_lazy_init", "k_row_items")}
    res = res_d.cpu().numpy().view(mp.RESULT_DTYPE)
    same = all(np.array_equal(res[k], res_eager[k]) for k in ("status", "path_len", "cost", "h", "relaxations"))
    Q = len(B.probs)
    if world > 1:   # whole-job value: all ranks' queries over the slowest rank's time
        import torch.distributed as dist
        t = torch.tensor([ms, float(same)], dtype=torch.float64, device="cuda")
        dist.all_reduce(t[:1], op=dist.ReduceOp.MAX)
        dist.all_reduce(t[1:], op=dist.ReduceOp.MIN)
        ms, same = float(t[0].item()), bool(t[1].item())
    return {"queries_per_s": world * Q * steps / (ms / 1e3), "ms_per_step": ms / steps, "rows_evaluated": rows[0],
            "rows_total": int(B.n.sum()), "same_results_as_eager": bool(same), "gpu_launches_per_step": launches / steps,
            "kernels_ms_per_step": {k: v[0] / steps for k, v in kern.items()},
            "search_launches_per_step": kern["k_search"][1] / steps}


def measure_mc(mp, B, betas, path_cap: int, trials: int, with_cpu: bool):
    """NEXT-4: Monte Carlo verification (Alg. 1 step 4,
    P:290) of the batch's feasible plans, `trials` trials each (Table 1 uses
    1000), in one k_mc launch; timed with the library's CUDA events on
    the launching stream (3 timed runs after 1 warm-up), outside the bench
    step.  The oracle times one trial per plan of a few plans on one core."""
    import torch
    from synth import mc_params
    mc = mc_params(trials=trials)
    rm = B.build()
    paths, res = B.search(rm, betas, path_capacity=path_cap)
    B.mc_verify(rm, paths, res, mc)
    torch.cuda.synchronize()
    mp.mpap_prof_reset()
    mp.mpap_prof_enable(True)
    runs = 3
    for k in range(runs):
        ok, mres, _ = B.mc_verify(rm, paths, res, mc, trial0=k * trials)
    mp.mpap_prof_enable(False)
    ms, n = mp.mpap_prof_read("k_mc")
    ms_plan, _ = mp.mpap_prof_read("k_mc_plan")
    rm.free()
    if mres is None:
        return {"plans": 0}
    t = (ms + ms_plan) / runs / 1e3
    steps = float(mres["steps"].sum()) * trials
    out = {"scope": "this rank's plans (per GPU)", "plans": int(ok.size), "trials_per_plan": trials,
           "ms_per_batch": (ms + ms_plan) / runs,
           "k_mc_ms": ms / max(n, 1), "trials_per_s": ok.size * trials / t, "trial_steps_per_s": steps / t,
           "p_hat_mean": float(mres["p_hat"].mean()), "fix_fraction": float(mres["fixes"].sum() / max(steps, 1)),
           "params": {k: mc[k] for k in ("sigma_imu", "sigma_vis", "delta", "k_p", "k_d", "u_max")}}
    if with_cpu:
        import oracle
        oracle.build()
        t0 = time.perf_counter()
        nt = 0
        for e in ok[:4]:
            path = paths[e][: res["path_len"][e]]
            for tr in range(8):
                oracle.mc_trial(B.probs[e], path, mc, tr)
                nt += 1
        dt = time.perf_counter() - t0
        out["cpu_baseline"] = {"value": nt / dt, "unit": "trials/s", "cores": 1, "kind": "oracle",
                               "sample": f"{nt} trials of {min(4, ok.size)} plans (1 thread)"}
    return out


# Algorithmic FP64 operations per counted unit (+, -, *, /, sqrt, min/max,
# compare and FMA each = 1), read off the kernels' source.
# D = 3, double integrator, heading + MLP heuristic (the C5 workload).
def step_stats(ms: list) -> dict:
    """Median, min and p90 (nearest rank) of this rank's timed steps (SURVEY 8(d) timing)."""
    xs = sorted(ms)
    if not xs:
        return {}
    p90 = xs[min(len(xs) - 1, max(0, math.ceil(0.9 * len(xs)) - 1))]
    return {"median": round(statistics.median(xs), 3), "min": round(xs[0], 3), "p90": round(p90, 3)}


def fp64_ops(kernel: str, w: dict, D: int = 3) -> float:
    if kernel == "k_near":
        return 18 * w["pairs"] + 101 * w["prefilter_pass"] + 9 * w["bisect_iters"]
    if kernel == "k_collide":
        return (12 * D + 2 * D + 4) * w["coll_segs"] + 4 * D * w["coll_box_tests"] + 27 * w["edges"]
    if kernel == "k_heuristic":
        # per step: t, position (3 per axis), heading interpolation (2 x 3 + 1), |h|^2 (DH);
        # range test 2D + 1, FOV test 2 DH + 3, occlusion segment 6D (dl, 1/dl, segment box),
        # slab box test 4D; per free edge 40 (trajectory, stationary points, arc).  The
        # heading heuristics' view vector is horizontal: DH = 2 terms in |h|^2 and the FOV
        # dot product (the kernels skip the z term, an exact zero)
        DH = 2
        per_step = 1 + 3 * D + 7 + DH
        return (per_step * w["steps"] + (2 * D + 1) * w["range_tests"] + (2 * DH + 3) * w["fov_tests"]
                + 6 * D * w["occl_segs"] + 4 * D * w["occl_box_tests"] + 40 * w["free_edges"])
    if kernel == "k_fold":
        # per step: increment 2, MLP 3-8-8-1 with ReLUs 128, speed (t, velocity 3D, |v|^2 D, sqrt) 14,
        # inputs 3 divisions, learned term 2, fold with running maxima 5; per free edge 36
        return (2 + 128 + 14 + 3 + 2 + 5) * w["steps"] + 36 * w["free_edges"]
    return 0.0


def committed_traffic(kernel: str, Q: int):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of `kernel` from
    the committed ncu --set full capture in the bench's launch configuration
    (profiles/traffic.json), or None."""
    try:
        t = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))
        e = t.get(kernel)
        if e and int(e.get("queries_per_gpu", -1)) == Q:
            return float(e["dram_bytes"])
    except Exception:
        pass
    return None


def roofline(kernel, ms, launches, work, B, res, peaks, peak_src, fp64=None, alg_bytes=None):
    """Achieved vs peak for the dominant kernel: algorithmic work per launch ÷
    its average launch duration (CUDA events on the launching stream)."""
    avg_s = (ms / max(launches, 1)) / 1e3
    if kernel == "k_search":
        simple = 16.0 * float(res["relaxations"].sum()) + 16.0 * float(res["labels_inserted"].sum())
        nbytes = float(alg_bytes["bytes"]) if alg_bytes else simple
        ach = nbytes / avg_s / 1e9 if avg_s > 0 else 0.0
        peak = float(peaks.get("hbm_gbs", FALLBACK_HBM_GBS))
        out = {"kernel": kernel, "bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s",
               "frac": ach / peak, "traffic": None, "peak_source": peak_src,
               "bytes_formula": "16 E_rows + 12 sum G + 8 F_reads + 16 L_ins (SURVEY 8(d), oracle counters)"
               if alg_bytes else "16 B per relaxation + 16 B per inserted label",
               "bytes_per_launch": nbytes}
        if alg_bytes:
            out["counters"] = alg_bytes
            out["simple_bytes_per_launch"] = simple
            out["simple_achieved"] = simple / avg_s / 1e9 if avg_s > 0 else 0.0
        return out
    ops = fp64_ops(kernel, work)
    mhz = float(peaks.get("sm_max_mhz", 1965.0))
    derived = SMS * FP64_LANES_PER_SM * mhz * 1e6 / 1e12
    peak = fp64["tops"] if fp64 else derived
    ach = ops / avg_s / 1e12 if avg_s > 0 else 0.0
    return {"kernel": kernel, "bound": "alu", "achieved": ach, "peak": peak,
            "unit": "T fp64 ops/s (one DFMA/DADD/DMUL instruction = one op)", "frac": ach / peak if peak else None,
            "traffic": None,
            "peak_source": "measured: FP64 issue-rate microbenchmark on this GPU (mpap_prof_fp64_peak, best of DFMA "
                           "and DADD streams)" if fp64 else f"derived ({peak_src} clock)",
            "peak_derived": derived,
            "peak_derived_source": f"{SMS} SMs x {FP64_LANES_PER_SM} FP64 lanes x {mhz:.0f} MHz",
            "ops_per_launch": ops, "work": {k: int(v) for k, v in work.items()}}


if __name__ == "__main__":
    sys.exit(main())
