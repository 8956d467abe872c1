"""NEXT-1 part i measurement: single query, eager build + search vs lazy build
(Near + Cost only) + lazy search (rows evaluated on first expansion), host
wall time around the synchronous C-ABI calls (each call synchronises), after
one warm-up; the lazy result is checked bit-identical to the eager one.

    python tools/bench_lazy.py [--configs c3,c4] [--reps 3] > gpurun_out/lazy.jsonl
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="c3,c4")
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    import torch
    import build_ext
    build_ext.build()
    import paper_1705_02408_b200 as mp
    from paper_1705_02408_b200.problem import build_problem, search_problem
    from synth import load_config, make_problem
    for name in args.configs.split(","):
        cfg = load_config(name)
        prob = make_problem(cfg)
        betas = [float(b) for b in cfg["betas"][:2]]
        for beta in betas:
            rows = {}
            for mode in ("eager", "lazy"):
                ts = []
                for rep in range(args.reps + 1):
                    torch.cuda.synchronize()
                    t0 = time.perf_counter()
                    rm = build_problem(prob, lazy_edges=(mode == "lazy"))
                    t1 = time.perf_counter()
                    r = search_problem(rm, prob, beta)
                    t2 = time.perf_counter()
                    ev = mp.mpap_roadmap_rows_evaluated(rm)
                    rm.free()
                    if rep:
                        ts.append((t1 - t0, t2 - t1))
                rows[mode] = {"build_ms": 1e3 * float(np.median([a for a, _ in ts])),
                              "search_ms": 1e3 * float(np.median([b for _, b in ts])),
                              "rows_evaluated": ev, "status": r["status"], "waves": r["waves"],
                              "path": r["path"].tolist(), "cost": float(r["cost"])}
                rows[mode]["total_ms"] = rows[mode]["build_ms"] + rows[mode]["search_ms"]
            assert rows["eager"]["path"] == rows["lazy"]["path"] and rows["eager"]["cost"] == rows["lazy"]["cost"]
            for m in rows.values():
                m.pop("path")
            print(json.dumps({"config": name, "n": prob.n, "beta": beta, **rows,
                              "speedup": rows["eager"]["total_ms"] / rows["lazy"]["total_ms"]}), flush=True)


if __name__ == "__main__":
    main()
