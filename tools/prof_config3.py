"""Config-3 posterior variance throughput (unequal n, lattice B4, d = 8): seconds for Q queries.
python tools/prof_config3.py [Q] [--profile]"""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_2603_16014_b200 import configs  # noqa: E402
from paper_2603_16014_b200.fast_gram import Model  # noqa: E402

Q = int(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1].isdigit() else 2048
inst = configs.make(3, n_test=Q)
M = Model(inst.design)
M.set_y(inst.y)
M.nll(inst.hyper, grad=False)
M.posterior_var(0, inst.X_test[:8])
if "--profile" in sys.argv:
    M.profile(True)
t0 = time.perf_counter()
v = M.posterior_var(0, inst.X_test[:Q])
dt = time.perf_counter() - t0
print(f"posterior_var {Q} queries: {dt:.3f} s ({1e6 * dt / Q:.1f} us/query), mean {np.mean(v):.6e}")
if "--profile" in sys.argv:
    for k, (ms, n) in M.profile_read().items():
        print(f"  {k:16s} {ms:9.2f} ms x {n}")
