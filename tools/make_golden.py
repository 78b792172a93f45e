#!/usr/bin/env python3
"""Generate tests/golden/*.npz from the reference library itself (oracle/_ref).

Each fixture stores the seeded design + hyperparameters + observations and the
reference's outputs through its own API (build_spectrum, invert_and_logdet, solve,
gram_matvec, trace_inverse, extract_pi_h, loss_value / tau / c, posterior_mean_batch,
posterior_cov, multitask_cubature).  Run in the container where /root/reference exists:
    python tools/make_golden.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import ref  # noqa: E402
from paper_2603_16014_b200 import configs  # noqa: E402
from paper_2603_16014_b200.designs import (DIGITAL, LATTICE, Hyper, digital_design, lattice_design,  # noqa: E402
                                           normal, uniform01)

OUT = os.path.join(ROOT, "tests", "golden")


def cases():
    for kind, mk in ((LATTICE, lattice_design), (DIGITAL, digital_design)):
        for m in ([3], [3, 2], [3, 2, 1], [2, 2, 2], [6, 6], [7, 4, 4, 2]):
            L, d = len(m), 2
            dz = mk(d, m, seed=1000 + len(m) * 10 + m[0])
            u = uniform01(77, 1 + kind, np.arange(64))
            hp = Hyper(gamma=float(np.exp(2 * u[0] - 0.5)), eta=np.exp(1.5 * u[1:1 + d] - 1.0),
                       B=(1.2 * (u[10:10 + L] - 0.5)).reshape(L, 1), t=0.05 + 0.5 * u[20:20 + L],
                       xi=1e-4 * (1 + u[30:30 + L]), si_alpha=1 + (m[0] % 2),
                       b=tuple(float(v) for v in np.exp(u[40:44] - 0.5)))
            y = normal(5, 6 + kind, np.arange(dz.N))
            yield f"{'lat' if kind == LATTICE else 'dig'}_{'-'.join(map(str, m))}", dz, hp, y
    c1 = configs.make(1, m=[7, 7], n_test=32)
    yield "config1_m7", c1.design, c1.hyper, c1.y
    c2 = configs.make(2, m=[6, 6, 6])
    yield "config2_m6", c2.design, c2.hyper, c2.y
    c3 = configs.make(3, m=[7, 5, 4, 2], n_test=8)
    yield "config3_small", c3.design, c3.hyper, c3.y


def save(name, dz, hp, y):
    b = normal(3, 2, np.arange(dz.N))
    lam = ref.build_spectrum(dz, hp)
    x, kb, logdet, tr, Pi = ref.invert_solve(dz, hp, b)
    model = ref.Model(dz, hp, y)
    nll = model.loss(0)
    st = model.state()
    X = uniform01(60, 0, np.arange(16 * dz.d)).reshape(16, dz.d)
    pm = np.stack([model.posterior_mean(t, X) for t in range(dz.L)])
    pv = np.array([[model.posterior_cov(t, X[q], t, X[q]) for q in range(4)] for t in range(dz.L)])
    mu, S = model.cubature()
    np.savez_compressed(
        os.path.join(OUT, name + ".npz"), kind=dz.kind, d=dz.d, m=np.array(dz.m), shift_bits=dz.shift_bits,
        g=dz.g if dz.g is not None else np.zeros(0, np.uint64), n_max=dz.n_max,
        columns=dz.columns if dz.columns is not None else np.zeros((0, 0), np.uint64), gamma=hp.gamma, eta=hp.eta,
        B=hp.B, t=hp.t, xi=hp.xi, si_alpha=hp.si_alpha, bw=np.array(hp.b), y=y, b=b,
        lam=np.concatenate(lam), x=x, kb=kb, logdet=logdet, trace=tr, Pi=Pi, nll=nll, tau=st["tau"], c=st["c"],
        X=X, post_mean=pm, post_var=pv, cub_mu=mu, cub_Sigma=S)


def load(path):
    from paper_2603_16014_b200.designs import Design
    z = np.load(path)
    kind = int(z["kind"])
    dz = Design(kind, int(z["d"]), [int(v) for v in z["m"]], z["shift_bits"],
                g=z["g"] if kind == LATTICE else None, n_max=int(z["n_max"]),
                columns=z["columns"] if kind == DIGITAL else None)
    hp = Hyper(gamma=float(z["gamma"]), eta=z["eta"], B=z["B"], t=z["t"], xi=z["xi"], si_alpha=int(z["si_alpha"]),
               b=tuple(float(v) for v in z["bw"]))
    return dz, hp, z


if __name__ == "__main__":
    os.makedirs(OUT, exist_ok=True)
    for name, dz, hp, y in cases():
        save(name, dz, hp, y)
        print("wrote", name, dz.N)
