"""FP64 issue-rate microbenchmark (mpap_prof_fp64_peak): DFMA, DADD, DMUL
instructions per second on cuda:0, one JSON line (profiles/r02/fp64_peak.json)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

torch.cuda.set_device(0)
import paper_1705_02408_b200 as mp  # noqa: E402

out = {}
for kind in ("dfma", "dadd", "dmul"):
    ops, ms = mp.mpap_prof_fp64_peak(kind)
    out[kind] = {"ops_per_s": ops, "tops": ops / 1e12, "ms": ms}
out["device"] = torch.cuda.get_device_name(0)
out["sms"] = torch.cuda.get_device_properties(0).multi_processor_count
print(json.dumps(out))
