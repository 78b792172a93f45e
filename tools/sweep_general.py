"""Seeded random-shape sweep of every path (lattice / digital, equal / unequal n, T <= 8, d <= 16,
shared shifts, Walsh order weights) against the reference library, all models kept alive in one
process: NLL, coefficients (solve floor), posterior mean, cubature mean.
python tools/sweep_general.py [cases] [seed]"""
import sys

import numpy as np

sys.path.insert(0, ".")
from oracle import ref  # noqa: E402  (test infrastructure: the checker)
from paper_2603_16014_b200.designs import Hyper, digital_design, lattice_design, normal, uniform01  # noqa: E402
from paper_2603_16014_b200.fast_gram import Model  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 40
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 5)
bad, models = 0, []
for k in range(n):
    kind = int(rng.integers(0, 2))
    T = int(rng.integers(1, 9))
    d = int(rng.integers(1, 17))
    m0 = int(rng.integers(3, 15 if len(sys.argv) > 3 else 11))
    equal = rng.random() < 0.5
    m = [m0] * T if equal else sorted([int(rng.integers(max(1, m0 - 4), m0 + 1)) for _ in range(T)], reverse=True)
    seed = int(rng.integers(1, 10000))
    dz = (lattice_design if kind == 0 else digital_design)(d, m, seed=seed)
    for t in range(1, T):
        if rng.random() < 0.25:
            dz.shift_bits[t] = dz.shift_bits[0]
    b = [(0.0, 0.0, 0.0, 1.0), (0.5, 0.2, 0.1, 1.0), (1.0, 0.0, 0.0, 0.0)][int(rng.integers(0, 3))]
    u = uniform01(seed, 9, np.arange(40))
    hp = Hyper(gamma=1.1, eta=0.1 + 0.5 * u[:d], B=normal(seed, 4, np.arange(2 * T)).reshape(T, 2),
               t=0.3 + 0.3 * u[20:20 + T], xi=np.full(T, 1e-3), si_alpha=1 + int(rng.integers(0, 2)), b=b)
    y = normal(seed + 1, 6, np.arange(dz.N))
    tag = (kind, T, d, m, seed, b, hp.si_alpha)
    try:
        M = Model(dz, max_candidates=2)
        M.set_y(y)
        models.append(M)
        r = M.nll(hp, grad=False)
        rm = ref.Model(dz, hp, y)
        want = rm.loss(0)
        st = rm.state()
        assert abs(r["nll"] - want) <= max(1e-8 * dz.N, 1e-8 * abs(r["quad"])), ("nll", r["nll"], want)
        c = M.coefficients()
        assert np.linalg.norm(c - st["c"]) <= 1e-7 * np.linalg.norm(st["c"]), ("c", np.linalg.norm(c - st["c"]))
        X = uniform01(seed, 77, np.arange(4 * d)).reshape(4, d)
        pm, pw = M.posterior_mean(0, X), rm.posterior_mean(0, X)
        assert np.linalg.norm(pm - pw) <= 1e-7 * max(1.0, np.linalg.norm(pw)), ("pm", pm, pw)
        pv = M.posterior_var(0, X[:2])
        pvw = np.array([rm.posterior_cov(0, X[q], 0, X[q]) for q in range(2)])
        assert np.abs(pv - pvw).max() <= 1e-7 * max(1.0, np.abs(pvw).max()), ("pv", pv, pvw)
        mu, _ = M.cubature()
        mu_r, _ = rm.cubature()
        assert np.linalg.norm(mu - mu_r) <= 1e-7 * max(1.0, np.linalg.norm(mu_r)), ("mu", mu, mu_r)
        if equal:
            rg = M.nll(hp, grad=True)
            assert abs(rg["nll"] - r["nll"]) <= 1e-9 * max(1.0, abs(r["nll"])), ("grad-nll", rg["nll"], r["nll"])
    except Exception as e:  # noqa: BLE001
        bad += 1
        print("FAIL", k, tag, repr(e)[:240], flush=True)
        if "CudaError" in repr(e):
            break
print("done", n, "bad", bad)
