"""Tuning harness (not the contract bench): per-kernel and per-phase times of
the batched build + search for a shard of the C5 workload.

    MPAP_LIB=paper_1705_02408_b200/libmpap_b2_u2.so python tools/bench_build.py [Q] [reps]
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1705_02408_b200 as mp  # noqa: E402
from paper_1705_02408_b200.problem import Batch  # noqa: E402
from synth import load_config, make_problem  # noqa: E402


def main():
    Q = int(sys.argv[1]) if len(sys.argv) > 1 else 64
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    cfg = load_config("c5")
    B = Batch([make_problem(cfg, env_index=k) for k in range(Q)])
    dev = torch.device("cuda")
    s_d = torch.from_numpy(B.samples).to(dev)
    o_d = torch.from_numpy(B.obstacles).to(dev)
    f_d = torch.from_numpy(B.features).to(dev)
    paths = torch.zeros((Q, 512), dtype=torch.int32, device=dev)
    res = torch.zeros(Q * 48, dtype=torch.uint8, device=dev)
    betas = [float(cfg["betas"][1])] * Q
    for _ in range(2):
        rm = B.build(s_d, o_d, f_d)
        B.search(rm, betas, 512, paths, res)
        rm.free()
    torch.cuda.synchronize()
    mp.mpap_prof_reset()
    mp.mpap_prof_enable(True)
    ph = {"build": 0.0, "search": 0.0, "free": 0.0}
    for _ in range(reps):
        t0 = time.perf_counter()
        rm = B.build(s_d, o_d, f_d)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        B.search(rm, betas, 512, paths, res)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        work = mp.mpap_roadmap_work(rm)
        rm.free()
        torch.cuda.synchronize()
        t3 = time.perf_counter()
        ph["build"] += (t1 - t0) * 1e3 / reps
        ph["search"] += (t2 - t1) * 1e3 / reps
        ph["free"] += (t3 - t2) * 1e3 / reps
    mp.mpap_prof_enable(False)
    kern = {k: mp.mpap_prof_read(k)[0] / reps for k in mp.KERNELS}
    print(json.dumps({"lib": os.path.basename(mp.LIB_PATH), "Q": Q, "phase_ms": ph, "kernel_ms": kern,
                      "work": work}))


if __name__ == "__main__":
    main()
