"""NEXT-1 measurement: time mpap_roadmap_update (one box moved, or a few
features edited) against a full rebuild, on the C5 shard (64 envs) and on one
C5 environment.  CUDA events on the launching stream; prints JSON lines."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1705_02408_b200 as mp
from paper_1705_02408_b200.problem import Batch
from synth import load_config, make_problem


def timed(fn, reps=5):
    st = torch.cuda.current_stream()
    out = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record(st)
        r = fn()
        b.record(st)
        b.synchronize()
        out.append(a.elapsed_time(b))
    return float(np.median(out)), r


def main():
    cfg = load_config("c5")
    for Q in (1, 64):
        probs = [make_problem(cfg, env_index=e) for e in range(Q)]
        B = Batch(probs)
        t_build, _ = timed(lambda: B.build().free(), reps=3)
        rm = B.build()
        p = probs[0]
        d = p.pos_dim
        box0 = p.obstacles.copy()
        moved = box0.copy()
        moved[7, :d] += 0.25
        moved[7, d:] += 0.25
        state = {"k": 0}

        def move():
            state["k"] ^= 1
            return mp.mpap_roadmap_update(rm, 0, moved if state["k"] else box0, p.features)
        t_move, n_move = timed(move)
        f0 = p.features.copy()
        f1 = f0.copy()
        f1[:5] += 0.5

        def feats():
            state["k"] ^= 1
            return mp.mpap_roadmap_update(rm, 0, box0, f1 if state["k"] else f0)
        mp.mpap_roadmap_update(rm, 0, box0, f0)
        state["k"] = 0
        t_feat, n_feat = timed(feats)
        nnz = sum(mp.mpap_roadmap_info(rm, e)["nnz"] for e in range(Q))
        nnz0 = mp.mpap_roadmap_info(rm, 0)["nnz"]
        print(json.dumps({"envs": Q, "full_build_ms": round(t_build, 3), "nnz_total": nnz, "nnz_env0": nnz0,
                          "move_one_box": {"ms": round(t_move, 3), "edges_reevaluated": n_move},
                          "move_five_features": {"ms": round(t_feat, 3), "edges_reevaluated": n_feat}}), flush=True)
        rm.free()


if __name__ == "__main__":
    main()
