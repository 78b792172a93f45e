"""Config-4 geometry with cheap synthetic y (profiling aid only: y values do not change the
kernels' work).  python tools/prof_config4.py [reps]"""
import sys
import numpy as np
sys.path.insert(0, ".")
from paper_2603_16014_b200 import configs  # noqa: E402
from paper_2603_16014_b200.designs import lattice_design  # noqa: E402
from paper_2603_16014_b200.fast_gram import Model  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 2
dz = lattice_design(4, [26, 26], seed=404)
hp = configs.config4(m=[4, 4]).hyper
y = np.random.default_rng(0).standard_normal(dz.N)
M = Model(dz)
M.set_y(y)
for _ in range(reps):
    r = M.nll(hp, grad=True)
print("nll", r["nll"])
