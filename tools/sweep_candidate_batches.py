"""Candidate batches (candidate groups of K1/K3 + per-candidate finalize) == single evaluations on
seeded random digital shapes.  python tools/sweep_candidate_batches.py"""
import sys
import numpy as np
sys.path.insert(0, ".")
from paper_2603_16014_b200.designs import Hyper, digital_design, normal, uniform01
from paper_2603_16014_b200.fast_gram import Model
rng = np.random.default_rng(3)
bad = 0
for k in range(25):
    T, m, d, seed = int(rng.integers(1, 5)), int(rng.integers(8, 17)), int(rng.integers(1, 13)), int(rng.integers(1, 9999))
    dz = digital_design(d, [m] * T, seed=seed)
    y = normal(seed + 1, 6, np.arange(dz.N))
    cands = []
    for c in range(int(rng.integers(2, 20))):
        u = uniform01(seed + c, 9, np.arange(32))
        cands.append(Hyper(gamma=0.5 + u[30], eta=0.05 + u[:d], B=normal(seed + c, 4, np.arange(2 * T)).reshape(T, 2),
                           t=0.2 + 0.3 * u[16:16 + T], xi=np.full(T, 1e-5), b=(0.0, 0.0, 0.0, 1.0)))
    M = Model(dz, max_candidates=16)
    M.set_y(y)
    batch = M.nll_batch(cands, grad=True)
    for h, rb in zip(cands, batch):
        rs = M.nll(h, grad=True)
        ok = abs(rs["nll"] - rb["nll"]) <= 1e-12 * abs(rs["nll"]) and np.allclose(rs["deta"], rb["deta"], rtol=1e-11, atol=0)
        if not ok:
            bad += 1
            print("FAIL", (T, m, d, seed, len(cands)), rs["nll"], rb["nll"], flush=True)
            break
print("done bad", bad)
