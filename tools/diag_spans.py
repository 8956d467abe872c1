"""Diagnostic: per-step host and GPU spans of the C5 build (MPAP_DEBUG_TIMING)."""
import sys, time, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1705_02408_b200 as mp
from paper_1705_02408_b200.problem import Batch
from synth import load_config, make_problem
cfg = load_config("c5")
probs = [make_problem(cfg, env_index=e) for e in range(64)]
B = Batch(probs)
dev = torch.device("cuda:0")
s_d = torch.from_numpy(B.samples).to(dev); o_d = torch.from_numpy(B.obstacles).to(dev); f_d = torch.from_numpy(B.features).to(dev)
for it in range(int(sys.argv[1]) if len(sys.argv) > 1 else 12):
    mp.mpap_prof_reset(); mp.mpap_prof_enable(True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rm = B.build(s_d, o_d, f_d)
    t1 = time.perf_counter()
    rm.free()
    torch.cuda.synchronize()
    out = {k: mp.mpap_prof_read(k)[0] for k in ("k_near", "k_collide", "k_heuristic", "span_edges", "span_wait")}
    print(json.dumps({"it": it, "host_build_ms": (t1 - t0) * 1e3, **{k: round(v, 2) for k, v in out.items()}}), flush=True)
