"""C4 perception-bound sweep (BASELINE.json configs[3]: "perception bound sweep
(tight to inactive), single query stress on 1 B200"): beta_min by batched
refinement on the GPU, then the sweep {inf, 2, 1.5, 1.25, 1.1, 1.02} x beta_min
as single queries (whole-grid search) and as one batched launch.

    python tools/c4_sweep.py [config]
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1705_02408_b200 as mp  # noqa: E402
from paper_1705_02408_b200.problem import beta_sweep, build_problem, refine_beta_min, search_problem  # noqa: E402
from synth import load_config, make_problem  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c4"
    prob = make_problem(load_config(name))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rm = build_problem(prob)
    torch.cuda.synchronize()
    t_build = time.perf_counter() - t0
    r_inf = search_problem(rm, prob, float("inf"))
    t0 = time.perf_counter()
    lo, hi, rounds = refine_beta_min(rm, prob, hi=float(r_inf["h_peak"]) * 1.0001 + 1e-9, rel_tol=1e-3)
    t_ref = time.perf_counter() - t0
    factors = [None, 2.0, 1.5, 1.25, 1.1, 1.02]
    betas = [float("inf") if f is None else f * hi for f in factors]
    out = {"config": name, "n": prob.n, "build_s": t_build, "beta_min": hi, "beta_min_bracket": [lo, hi],
           "refine_rounds": rounds, "refine_s": t_ref, "single": []}
    for beta in betas:
        search_problem(rm, prob, beta)
        mp.mpap_prof_reset()
        mp.mpap_prof_enable(True)
        r = search_problem(rm, prob, beta)
        mp.mpap_prof_enable(False)
        ms, n = mp.mpap_prof_read("k_search")
        out["single"].append({"beta": beta, "status": r["status_str"], "cost": float(r["cost"]), "h": float(r["h"]),
                              "waves": r["waves"], "relaxations": r["relaxations"], "kernel_ms": ms / max(n, 1),
                              "edges_relaxed_per_s": r["relaxations"] / (ms / max(n, 1) / 1e3) if ms else None})
    beta_sweep(rm, prob, betas)
    mp.mpap_prof_reset()
    mp.mpap_prof_enable(True)
    _, res = beta_sweep(rm, prob, betas)
    mp.mpap_prof_enable(False)
    ms, n = mp.mpap_prof_read("k_search")
    out["batched_sweep"] = {"betas": len(betas), "kernel_ms": ms, "launches": n,
                            "relaxations": int(res["relaxations"].sum()),
                            "statuses": res["status"].tolist()}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
