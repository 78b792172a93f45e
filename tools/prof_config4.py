"""Config-4 geometry with cheap synthetic y (profiling aid only: y values do not change the
kernels' work).  python tools/prof_config4.py [reps] [--profile]
Prints the NLL, the median wall time per evaluation and (with --profile) per-kernel event times."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_2603_16014_b200 import configs  # noqa: E402
from paper_2603_16014_b200.designs import lattice_design  # noqa: E402
from paper_2603_16014_b200.fast_gram import Model  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1].isdigit() else 2
dz = lattice_design(4, [26, 26], seed=404)
hp = configs.config4(m=[4, 4]).hyper
y = np.random.default_rng(0).standard_normal(dz.N)
M = Model(dz)
M.set_y(y)
ts = []
for _ in range(reps):
    t0 = time.perf_counter()
    r = M.nll(hp, grad=True)
    ts.append(time.perf_counter() - t0)
print("nll", r["nll"], "wall_ms_med", 1e3 * float(np.median(ts[1:] if len(ts) > 1 else ts)))
if "--profile" in sys.argv:
    M.profile(True)
    for _ in range(reps):
        M.nll(hp, grad=True)
    for k, (ms, n) in M.profile_read().items():
        print(f"  {k:16s} {ms / max(n, 1):8.3f} ms x {n}")
