"""Calibrates the frozen perception bounds of a config:
beta_min = smallest beta (to 1e-3 relative) for which the oracle returns a
plan at the config's lambda; prints {inf, 1.25, 1.5, 2} x beta_min.
Calls only oracle/ and synth/.

    python tools/calibrate_beta.py c3 [env_index]
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
from synth import load_config, make_problem  # noqa: E402


def beta_min(rm, prob):
    r_inf = oracle.search(rm, prob, float("inf"))
    if r_inf["status"] != 0:
        return None, r_inf
    lo, hi = 0.0, float(r_inf["h_peak"])
    if oracle.search(rm, prob, 0.0)["status"] == 0:
        return 0.0, r_inf
    while hi - lo > 1e-3 * hi:
        mid = 0.5 * (lo + hi)
        if oracle.search(rm, prob, mid)["status"] == 0:
            hi = mid
        else:
            lo = mid
    return hi, r_inf


def main():
    name = sys.argv[1]
    env = int(sys.argv[2]) if len(sys.argv) > 2 else None
    prob = make_problem(load_config(name), env_index=env)
    rm = oracle.build_roadmap_parallel(prob)
    bm, r_inf = beta_min(rm, prob)
    print(f"{prob.name}: agnostic cost {r_inf['cost']} h {r_inf['h']} h_peak {r_inf['h_peak']}; beta_min {bm}")
    if bm is not None:
        for f in (1.02, 1.1, 1.25, 1.5, 2.0):
            r = oracle.search(rm, prob, f * bm)
            print(f"  {f:5.2f} x beta_min = {f * bm:.4f}: cost {r['cost']} h {r['h']} waves {r['waves']} "
                  f"relax {r['relaxations']}")


if __name__ == "__main__":
    main()
