"""Reproducer for the cross-model digital-fit failure fixed in model.cu (undersized d_work of the fused
path at small n): runs one model of shape "case 6" and then checks "case 11".  python tools/repro_pair.py ours6"""
import sys
import numpy as np
sys.path.insert(0, ".")
from oracle import ref
from paper_2603_16014_b200.designs import Hyper, digital_design, normal, uniform01
from paper_2603_16014_b200.fast_gram import Model

def inst(T, m, d, seed, shared, bi):
    dz = digital_design(d, [m] * T, seed=seed)
    for t in shared:
        dz.shift_bits[t] = dz.shift_bits[0]
    b = [(0.0, 0.0, 0.0, 1.0), (0.5, 0.2, 0.1, 1.0), (1.0, 0.0, 0.0, 0.0)][bi]
    u = uniform01(seed, 9, np.arange(32))
    hp = Hyper(gamma=1.2, eta=0.1 + u[:d], B=normal(seed, 4, np.arange(2 * T)).reshape(T, 2), t=0.2 + 0.3 * u[16:16 + T], xi=np.full(T, 1e-5), b=b)
    return dz, hp, normal(seed + 1, 6, np.arange(dz.N))

mode = sys.argv[1]
a = inst(4, 11, 10, 5991, [3], 0)
b = inst(3, 8, 12, 8347, [], 2)
if "ours6" in mode:
    M = Model(a[0], max_candidates=4); M.set_y(a[2]); print("6 ours", M.nll(a[1], grad=True)["nll"])
if "ref6" in mode:
    print("6 ref", ref.Model(*a).loss(0))
M2 = Model(b[0], max_candidates=4); M2.set_y(b[2]); print("11 ours", M2.nll(b[1], grad=True)["nll"])
print("11 ref", ref.Model(*b).loss(0))
