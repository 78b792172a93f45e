"""Reproducer for one digital-fit shape: T m d seed b_index [max_candidates grad]."""
import sys
import numpy as np
sys.path.insert(0, ".")
from oracle import ref
from paper_2603_16014_b200.designs import Hyper, digital_design, normal, uniform01
from paper_2603_16014_b200.fast_gram import Model
T, m, d, seed, b = [int(x) for x in sys.argv[1:5]] + [None]
b = [(0.0, 0.0, 0.0, 1.0), (0.5, 0.2, 0.1, 1.0), (1.0, 0.0, 0.0, 0.0)][int(sys.argv[5])]
dz = digital_design(d, [m] * T, seed=seed)
u = uniform01(seed, 9, np.arange(32))
hp = Hyper(gamma=1.2, eta=0.1 + u[:d], B=normal(seed, 4, np.arange(2 * T)).reshape(T, 2), t=0.2 + 0.3 * u[16:16 + T], xi=np.full(T, 1e-5), b=b)
y = normal(seed + 1, 6, np.arange(dz.N))
mc = int(sys.argv[6]) if len(sys.argv) > 6 else 1
grad = bool(int(sys.argv[7])) if len(sys.argv) > 7 else False
M = Model(dz, max_candidates=mc)
M.set_y(y)
want = ref.Model(dz, hp, y).loss(0)
for k in range(3):  # eager run, capture, replay
    r = M.nll(hp, grad=grad)
    print("ours", r["nll"], "ref", want, flush=True)
