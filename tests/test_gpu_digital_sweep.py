"""Seeded random shapes of the fused digital fit against the reference library, several models
alive in one process (regression: small n, whose generic geometry is single-pass, once gave the
fused path an undersized staging buffer — out-of-bounds writes that only showed as wrong NLLs of
LATER models).  The full 60-case sweep is tools/sweep_digital_fused.py."""
import numpy as np
import pytest

from paper_2603_16014_b200.designs import Hyper, digital_design, normal, uniform01

pytestmark = pytest.mark.gpu


def _cases(n, seed=99):
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(n):
        T, m, d, s = int(rng.integers(1, 5)), int(rng.integers(6, 15)), int(rng.integers(1, 17)), int(rng.integers(1, 10000))
        shared = [t for t in range(1, T) if rng.random() < 0.3]
        out.append((T, m, d, s, shared, int(rng.integers(0, 3))))
    return out


def test_digital_random_shapes_sequential(ref):
    from paper_2603_16014_b200.fast_gram import Model
    models = []  # keep every model alive: stray writes would land in a live neighbour
    for T, m, d, seed, shared, bi in _cases(16):
        dz = digital_design(d, [m] * T, seed=seed)
        for t in shared:
            dz.shift_bits[t] = dz.shift_bits[0]
        b = [(0.0, 0.0, 0.0, 1.0), (0.5, 0.2, 0.1, 1.0), (1.0, 0.0, 0.0, 0.0)][bi]
        u = uniform01(seed, 9, np.arange(32))
        hp = Hyper(gamma=1.2, eta=0.1 + u[:d], B=normal(seed, 4, np.arange(2 * T)).reshape(T, 2),
                   t=0.2 + 0.3 * u[16:16 + T], xi=np.full(T, 1e-5), b=b)
        y = normal(seed + 1, 6, np.arange(dz.N))
        M = Model(dz, max_candidates=4)
        M.set_y(y)
        models.append(M)
        r = M.nll(hp, grad=True)
        want = ref.Model(dz, hp, y).loss(0)
        assert abs(r["nll"] - want) <= max(1e-8 * dz.N, 1e-9 * abs(r["quad"])), (T, m, d, seed, r["nll"], want)
        cands = [hp, hp.replace(eta=hp.eta * 1.3), hp.replace(gamma=0.8)]
        for h, rb in zip(cands, M.nll_batch(cands, grad=True)):
            rs = M.nll(h, grad=True)
            assert rs["nll"] == rb["nll"] and np.array_equal(rs["deta"], rb["deta"])


def test_all_paths_random_shapes(ref):
    """tools/sweep_general.py's checks on 30 seeded shapes (lattice / digital, equal / unequal n,
    T <= 8, d <= 16, shared shifts): NLL, coefficients, posterior mean / variance, cubature."""
    import subprocess
    import sys
    out = subprocess.run([sys.executable, "tools/sweep_general.py", "30", "31"], capture_output=True, text=True,
                         timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    assert "bad 0" in out.stdout, out.stdout[-3000:]
