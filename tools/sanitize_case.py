"""Small workload for compute-sanitizer (racecheck / synccheck / memcheck):
the three search team kinds and the build kernels on small roadmaps, each
result compared with the CPU oracle.

    compute-sanitizer --tool racecheck python tools/sanitize_case.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_1705_02408_b200 as mp  # noqa: E402
from paper_1705_02408_b200.problem import Batch, build_problem, search_problem  # noqa: E402
from synth import load_config, make_problem  # noqa: E402

torch.cuda.set_device(0)
ok = True
c1 = make_problem(load_config("c1"))
rm = build_problem(c1)
o1 = oracle.build_roadmap(c1)
for beta in (float("inf"), 0.2174):
    g = search_problem(rm, c1, beta)                     # whole-grid team (cooperative launch)
    o = oracle.search(o1, c1, beta)
    ok &= g["status"] == o["status"] and g["path"].tolist() == o["path"].tolist()
rm.free()
cfg = load_config("c3")
cfg["n_samples"] = 300
probs = [make_problem(cfg), make_problem(dict(cfg, env_seed=11))]
B = Batch(probs)
rm = B.build()
orms = [oracle.build_roadmap(p) for p in probs]
betas = [float("inf"), 6.0, 4.0, 3.0]
envs = np.repeat(np.arange(2, dtype=np.int32), len(betas))
bq = np.tile(np.asarray(betas), 2)
for mode in ("MPAP_SEARCH_NO_GRID", "MPAP_SEARCH_CTA"):      # cluster team, CTA team
    os.environ[mode] = "1"
    paths, res = B.search(rm, bq, path_capacity=256, envs=envs)
    del os.environ[mode]
    for q in range(len(envs)):
        o = oracle.search(orms[envs[q]], probs[envs[q]], bq[q])
        ok &= int(res[q]["status"]) == o["status"]
        if o["status"] == 0:
            ok &= paths[q, : res[q]["path_len"]].tolist() == o["path"].tolist()
rm.free()
print("sanitize case", "OK" if ok else "MISMATCH", mp.mpap_search_launches(), flush=True)
sys.exit(0 if ok else 1)
