"""One roadmap build + `reps` single queries (whole-grid search) of a config
at one bound -- the short command the search ncu captures profile.

    python tools/one_search.py c4 8.8245 [reps]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1705_02408_b200 as mp  # noqa: E402
from paper_1705_02408_b200.problem import build_problem, search_problem  # noqa: E402
from synth import load_config, make_problem  # noqa: E402

name, beta = sys.argv[1], float(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
torch.cuda.set_device(0)
prob = make_problem(load_config(name))
rm = build_problem(prob)
mp.mpap_prof_reset()
mp.mpap_prof_enable(True)
for _ in range(reps):
    r = search_problem(rm, prob, beta)
mp.mpap_prof_enable(False)
ms, n = mp.mpap_prof_read("k_search")
print(json.dumps({"config": name, "beta": beta, "status": r["status_str"], "waves": r["waves"],
                  "relaxations": r["relaxations"], "kernel_ms": ms / max(n, 1), "teams": mp.mpap_search_launches()}))
rm.free()
