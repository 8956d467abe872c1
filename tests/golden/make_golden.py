"""Writes tests/golden/*.json: oracle results at BASELINE.json's full sizes.

Calls only oracle/ (and the synth/ input generators); nothing here touches
the CUDA path.  The GPU parity tests compare libmpap.so against these stored
oracle outputs, because the full-size oracle build takes minutes of CPU.

    python tests/golden/make_golden.py [c3] [c5] [c4] [c5_bench] [c5_all] [c4_tight]

c5_bench: the bench's rank-0 shard (C5 environments 0..63) at four bounds
each -- the 64-query batch the bench times (beta = configs/c5.json betas[1])
and a 256-query batch -- with CSR digests of every environment.
"""
from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from synth import load_config, make_problem  # noqa: E402

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from digest import csr_digests  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def f32hex(x) -> str:
    return np.float32(x).tobytes().hex()


def run_one(prob, betas, procs):
    t = time.time()
    rm = oracle.build_roadmap_parallel(prob, procs)
    tb = time.time() - t
    free = rm["coll"] == 0
    out = {"name": prob.name, "n": int(prob.n), "nnz": int(len(rm["dst"])), "nnz_free": int(free.sum()),
           "w_sum": float(rm["w"].astype(np.float64).sum()), "s_sum": float(rm["s"][free].astype(np.float64).sum()),
           "c_sum": float(rm["c"][free].astype(np.float64).sum()), "oracle_build_s": tb,
           "digests": csr_digests(rm), "searches": []}
    for beta in betas:
        t = time.time()
        r = oracle.search(rm, prob, beta)
        out["searches"].append({
            "beta": beta if np.isfinite(beta) else "inf", "status": r["status"], "path": r["path"].tolist(),
            "cost": f32hex(r["cost"]), "h": f32hex(r["h"]), "h_peak": f32hex(r["h_peak"]), "waves": r["waves"],
            "relaxations": r["relaxations"], "labels_inserted": r["labels_inserted"],
            "wave_counters": r["wave_counters"].tolist(), "e_rows": r["e_rows"],
            "oracle_search_s": time.time() - t,
        })
        print(prob.name, beta, r["status_str"], r["cost"], r["h"], r["waves"], r["relaxations"], flush=True)
    return out


def main(argv):
    procs = os.cpu_count() or 1
    which = argv or ["c3", "c5"]
    if "c3" in which:
        cfg = load_config("c3")
        prob = make_problem(cfg)
        res = run_one(prob, [float(b) if b != "inf" else float("inf") for b in cfg["golden_betas"]], procs)
        json.dump(res, open(os.path.join(HERE, "c3_full.json"), "w"), indent=1)
    if "c5" in which:
        cfg = load_config("c5")
        envs = []
        for k in range(cfg["golden_envs"]):
            prob = make_problem(cfg, env_index=k)
            envs.append(run_one(prob, [float(b) if b != "inf" else float("inf") for b in cfg["golden_betas"]],
                                procs))
        json.dump({"envs": envs}, open(os.path.join(HERE, "c5_full.json"), "w"), indent=1)
    if "c5_bench" in which:
        cfg = load_config("c5")
        betas = [float(cfg["betas"][1]), float("inf"), 2.2, 3.2]
        envs = []
        for k in range(int(cfg["queries_per_gpu"])):
            prob = make_problem(cfg, env_index=k)
            envs.append(run_one(prob, betas, procs))
        json.dump({"betas": ["inf" if not np.isfinite(b) else b for b in betas], "envs": envs},
                  open(os.path.join(HERE, "c5_bench.json"), "w"), indent=None)
    if "c5_all" in which:
        # every C5 environment at the bench bound (the parity gate of every
        # rank of the weak-scaling bench, and of a 512-query single-GPU run);
        # environments of c5_bench.json are taken from there (same oracle run)
        cfg = load_config("c5")
        beta = float(cfg["betas"][1])
        have = {}
        bench_path = os.path.join(HERE, "c5_bench.json")
        if os.path.exists(bench_path):
            bj = json.load(open(bench_path))
            k0 = [float("inf") if b == "inf" else float(b) for b in bj["betas"]].index(beta)
            for env in bj["envs"]:
                e = dict(env)
                e["searches"] = [env["searches"][k0]]
                have[env["name"]] = e
        envs = []
        for k in range(int(cfg["n_queries"])):
            prob = make_problem(cfg, env_index=k)
            envs.append(have.get(prob.name) or run_one(prob, [beta], procs))
            if k % 16 == 15:   # checkpoint (the full run takes over an hour on 8 cores)
                json.dump({"beta": beta, "envs": envs}, open(os.path.join(HERE, "c5_all.json"), "w"))
        json.dump({"beta": beta, "envs": envs}, open(os.path.join(HERE, "c5_all.json"), "w"))
    if "c4_tight" in which:
        # C4 at the tightest bound of its sweep (1.02 beta_min): 105 waves, 2e8
        # relaxations, staircases of thousands of plans -- the large-node merge
        # paths of the search.  The literal oracle search takes ~35 min.
        cfg = load_config("c4")
        prob = make_problem(cfg)
        res = run_one(prob, [float(cfg["betas"][-1])], procs)
        json.dump(res, open(os.path.join(HERE, "c4_tight.json"), "w"), indent=1)
    if "c4" in which:
        cfg = load_config("c4")
        prob = make_problem(cfg)
        res = run_one(prob, [float(b) if b != "inf" else float("inf") for b in cfg["golden_betas"]], procs)
        json.dump(res, open(os.path.join(HERE, "c4_full.json"), "w"), indent=1)


if __name__ == "__main__":
    main(sys.argv[1:])
