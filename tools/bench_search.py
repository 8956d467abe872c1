"""Single-query and batched search timing on BASELINE configs (tuning aid):
builds each config's roadmap once, then times mpap_search per beta with CUDA
events (device-resident roadmap, host result), reports relaxations/s.

    python tools/bench_search.py [c1 c2 c3 c4] [--reps N]
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1705_02408_b200 as mp  # noqa: E402
from paper_1705_02408_b200.problem import build_problem, search_problem  # noqa: E402
from synth import load_config, make_problem  # noqa: E402


def main():
    args = sys.argv[1:]
    reps = 5
    if "--reps" in args:
        k = args.index("--reps")
        reps = int(args[k + 1])
        del args[k:k + 2]
    names = args or ["c1", "c2", "c3", "c4"]
    for name in names:
        cfg = load_config(name)
        prob = make_problem(cfg)
        t0 = time.perf_counter()
        rm = build_problem(prob)
        torch.cuda.synchronize()
        tb = time.perf_counter() - t0
        info = mp.mpap_roadmap_info(rm)
        betas = [float("inf") if b == "inf" else float(b) for b in cfg.get("betas", ["inf"])]
        for beta in betas:
            r = search_problem(rm, prob, beta)
            mp.mpap_prof_reset()
            mp.mpap_prof_enable(True)
            t0 = time.perf_counter()
            for _ in range(reps):
                r = search_problem(rm, prob, beta)
            wall = (time.perf_counter() - t0) / reps
            mp.mpap_prof_enable(False)
            ks, kn = mp.mpap_prof_read("k_search")
            kms = ks / max(kn, 1)
            print(json.dumps({"config": name, "n": info["n"], "nnz": info["nnz"], "build_s": round(tb, 3),
                              "beta": beta, "status": r["status_str"], "cost": float(r["cost"]), "h": float(r["h"]),
                              "waves": r["waves"], "relaxations": r["relaxations"],
                              "kernel_ms": round(kms, 3), "call_ms": round(wall * 1e3, 3),
                              "edges_relaxed_per_s": r["relaxations"] / (kms / 1e3) if kms > 0 else None}))
        rm.free()


if __name__ == "__main__":
    main()
