"""Config-5 candidate sweep (256 candidates, 64 per batch): wall time per sweep and per-kernel
event times.  python tools/prof_config5.py [reps] [--profile]"""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_2603_16014_b200 import configs  # noqa: E402
from paper_2603_16014_b200.fast_gram import Model  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1].isdigit() else 3
inst = configs.make(5)
mc = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2].isdigit() else 64
M = Model(inst.design, max_candidates=mc)
M.set_y(inst.y)
ts = []
for _ in range(reps):
    t0 = time.perf_counter()
    res = M.nll_batch(inst.candidates, grad=True)
    ts.append(time.perf_counter() - t0)
print("nll[0]", res[0]["nll"], "deta[0]", res[0]["deta"][:3], "sweep_ms_med", 1e3 * float(np.median(ts[1:] if len(ts) > 1 else ts)))
if "--profile" in sys.argv:
    M.profile(True)
    M.nll_batch(inst.candidates, grad=True)
    for k, (ms, n) in M.profile_read().items():
        print(f"  {k:16s} {ms:9.3f} ms total x {n}")
