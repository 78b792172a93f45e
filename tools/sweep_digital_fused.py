"""Seeded random-shape sweep of the fused digital fit (K1-K3) against the reference library:
NLL / logdet within 1e-8 N (or the solve floor), batched candidate groups == single evaluations.
python tools/sweep_digital_fused.py [cases]"""
import sys

import numpy as np

sys.path.insert(0, ".")
from oracle import ref  # noqa: E402  (test infrastructure: the checker)
from paper_2603_16014_b200.designs import Hyper, digital_design, normal, uniform01  # noqa: E402
from paper_2603_16014_b200.fast_gram import Model  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 40
only = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else None
rng = np.random.default_rng(99)
bad = 0
for k in range(n):
    T = int(rng.integers(1, 5))
    m = int(rng.integers(6, 15))
    d = int(rng.integers(1, 17))
    seed = int(rng.integers(1, 10000))
    dz = digital_design(d, [m] * T, seed=seed)
    for t in range(1, T):
        if rng.random() < 0.3:
            dz.shift_bits[t] = dz.shift_bits[0]
    b = [(0.0, 0.0, 0.0, 1.0), (0.5, 0.2, 0.1, 1.0), (1.0, 0.0, 0.0, 0.0)][int(rng.integers(0, 3))]
    u = uniform01(seed, 9, np.arange(32))
    hp = Hyper(gamma=1.2, eta=0.1 + u[:d], B=normal(seed, 4, np.arange(2 * T)).reshape(T, 2), t=0.2 + 0.3 * u[16:16 + T],
               xi=np.full(T, 1e-5), b=b)
    y = normal(seed + 1, 6, np.arange(dz.N))
    if only is not None and k not in only:
        continue
    try:
        M = Model(dz, max_candidates=4)
        M.set_y(y)
        r = M.nll(hp, grad=True)
        want = ref.Model(dz, hp, y).loss(0)
        assert abs(r["nll"] - want) <= max(1e-8 * dz.N, 1e-9 * abs(r["quad"])), (r["nll"], want)
        cands = [hp, hp.replace(eta=hp.eta * 1.3), hp.replace(gamma=0.8)]
        batch = M.nll_batch(cands, grad=True)
        for h, rb in zip(cands, batch):
            rs = M.nll(h, grad=True)
            assert rs["nll"] == rb["nll"] and np.array_equal(rs["deta"], rb["deta"])
    except Exception as e:  # noqa: BLE001
        bad += 1
        try:
            ref_out = ref.Model(dz, hp, y).loss(0)
        except Exception as e2:  # noqa: BLE001
            ref_out = repr(e2)[:80]
        print("FAIL", k, (T, m, d, seed, b), repr(e)[:200], "| reference:", ref_out, flush=True)
        if "CudaError" in repr(e):
            break
print("done", n, "bad", bad)
