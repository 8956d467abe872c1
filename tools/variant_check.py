"""Tuning harness for build-kernel variants (MPAP_LIB=<variant .so>): the
bench's 64-environment C5 shard, per-kernel CUDA-event times over `reps`
batched builds, and the CSR digests of every environment against the
oracle's goldens (tests/golden/c5_bench.json).  One JSON line.

    MPAP_LIB=paper_1705_02408_b200/libmpap_v11.so python tools/variant_check.py [reps]
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
import torch  # noqa: E402

import paper_1705_02408_b200 as mp  # noqa: E402
from digest import csr_digests  # noqa: E402
from paper_1705_02408_b200.problem import Batch  # noqa: E402
from synth import load_config, make_problem  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
gold = json.load(open(os.path.join(ROOT, "tests", "golden", "c5_bench.json")))
cfg = load_config("c5")
B = Batch([make_problem(cfg, env_index=k) for k in range(len(gold["envs"]))])
dev = torch.device("cuda")
s_d = torch.from_numpy(B.samples).to(dev)
o_d = torch.from_numpy(B.obstacles).to(dev)
f_d = torch.from_numpy(B.features).to(dev)
rm = B.build(s_d, o_d, f_d)
bad = [e for e in range(len(gold["envs"])) if csr_digests(mp.mpap_roadmap_export(rm, e)) != gold["envs"][e]["digests"]]
rm.free()
torch.cuda.synchronize()
mp.mpap_prof_reset()
mp.mpap_prof_enable(True)
for _ in range(reps):
    rm = B.build(s_d, o_d, f_d)
    work = mp.mpap_roadmap_work(rm)
    rm.free()
torch.cuda.synchronize()
mp.mpap_prof_enable(False)
print(json.dumps({"lib": os.path.basename(mp.LIB_PATH), "digests_ok": not bad, "bad_envs": bad[:8],
                  "ms": {k: round(mp.mpap_prof_read(k)[0] / reps, 3) for k in mp.KERNELS if k != "k_search"},
                  "work": {k: int(v) for k, v in work.items()}}), flush=True)
