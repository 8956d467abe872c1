"""NEXT-4 demonstration: Monte Carlo verification (Alg. 1 step 4) of
perception-agnostic (beta = inf) vs perception-aware (beta = config) plans on
the C5 environments -- the comparison of the paper's Table 1, on our
synthetic workload.  Per-trial max localisation errors come from one batched
k_mc launch per beta; p_hat is reported for several bounds delta.

    python tools/mc_sweep.py [--envs 64] [--trials 1000] > gpurun_out/mc_sweep.json
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--envs", type=int, default=64)
    ap.add_argument("--trials", type=int, default=1000)
    ap.add_argument("--config", default="c5")
    args = ap.parse_args()
    import torch
    import build_ext
    build_ext.build()
    from paper_1705_02408_b200.problem import Batch
    from synth import load_config, make_problem, mc_params
    cfg = load_config(args.config)
    probs = [make_problem(cfg, env_index=k) for k in range(args.envs)]
    B = Batch(probs)
    rm = B.build()
    mc = mc_params(trials=args.trials)
    out = {"config": args.config, "envs": args.envs, "trials": args.trials, "mc": mc, "betas": {}}
    both = None
    per = {}
    for beta in (float("inf"), float(cfg["betas"][1])):
        paths, res = B.search(rm, [beta] * args.envs, path_capacity=512)
        ok, mres, me = B.mc_verify(rm, paths, res, mc, per_trial=True)
        per[beta] = dict(zip(ok.tolist(), me))
        both = set(ok.tolist()) if both is None else both & set(ok.tolist())
        out["betas"][str(beta)] = {"feasible": int(ok.size), "mean_cost": float(res["cost"][ok].mean()),
                                   "mean_h": float(res["h"][ok].mean())}
    torch.cuda.synchronize()
    envs = sorted(both)
    out["common_envs"] = len(envs)
    for beta, d in per.items():
        e = np.stack([d[k] for k in envs])
        row = out["betas"][str(beta)]
        row["median_max_err"] = float(np.median(e))
        row["p99_max_err"] = float(np.percentile(e, 99))
        row["p_hat"] = {str(dl): float((e >= dl).mean()) for dl in (0.1, 0.15, 0.2, 0.3, 0.5)}
    rm.free()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
