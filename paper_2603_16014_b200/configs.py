"""The five BASELINE.json workloads as seeded synthetic instances.

No public dataset is involved: every config is a closed-form synthetic target on
seeded designs (BASELINE.json ``configs``; SURVEY.md §8d "Synthetic inputs").
``m_override`` shrinks a config to test size while keeping T, d, kernel and
hyperparameter structure, so parity tests run the same code path as the bench.
"""
from __future__ import annotations

import dataclasses
from typing import List, Optional

import numpy as np

from .designs import (DIGITAL, LATTICE, Design, Hyper, bits_to_frac, digital_design,
                      lattice_design, normal, uniform01)

NOISE_STD = 1e-3  # N(0, 1e-6)


@dataclasses.dataclass
class Instance:
    name: str
    design: Design
    hyper: Hyper
    y: np.ndarray  # internal order, length N
    outputs: tuple
    X_test: Optional[np.ndarray] = None  # [Q, d] test points
    candidates: Optional[List[Hyper]] = None  # config 5


def _targets(design: Design, f, seed: int) -> np.ndarray:
    ys = []
    for l in range(design.L):
        x = design.points(l)
        yl = f(x, l) + NOISE_STD * normal(seed, 0x0B5 + l, np.arange(x.shape[0]))
        ys.append(yl)
    return np.concatenate(ys)


def _y_sines(design, seed):  # configs 1 and 4
    return _targets(design, lambda x, t: (1 + 0.3 * t) * np.sin(2 * np.pi * x).sum(axis=1), seed)


def _y_prod(design, seed):  # configs 2 and 5
    j = np.arange(1, design.d + 1)
    return _targets(design, lambda x, t: np.prod(1 + (x - 0.5) / j, axis=1) * (1 + 0.2 * t), seed)


def _y_exp(design, seed):  # config 3
    j = np.arange(1, design.d + 1)
    return _targets(design, lambda x, t: np.exp(-(x / (j + 1)).sum(axis=1)) * (1 + 0.1 * t), seed)


def config1(seed: int = 101, m: Optional[List[int]] = None, n_test: int = 4096) -> Instance:
    T, d = 2, 2
    m = m or [10] * T
    dz = lattice_design(d, m, seed)
    w = normal(seed, 0x77, np.arange(T)).reshape(T, 1)
    hp = Hyper(gamma=1.0, eta=np.ones(d), B=w, t=np.full(T, 0.5), xi=np.full(T, 1e-8), si_alpha=1)
    X = uniform01(seed, 0x7E57, np.arange(n_test * d)).reshape(n_test, d)
    return Instance("config1", dz, hp, _y_sines(dz, seed), ("c", "logdet", "nll", "posterior_mean"), X_test=X)


def config2(seed: int = 202, m: Optional[List[int]] = None) -> Instance:
    T, d = 3, 5
    m = m or [16] * T
    dz = digital_design(d, m, seed)
    B = normal(seed, 0x77, np.arange(T * 2)).reshape(T, 2)
    t = 0.1 + 0.5 * uniform01(seed, 0x78, np.arange(T))
    hp = Hyper(gamma=1.0, eta=1.0 / np.arange(1, d + 1), B=B, t=t, xi=np.full(T, 1e-8), b=(0.0, 0.0, 0.0, 1.0))
    return Instance("config2", dz, hp, _y_prod(dz, seed), ("nll", "grad_eta", "grad_w", "grad_v"))


def config3(seed: int = 303, m: Optional[List[int]] = None, n_test: int = 1 << 14) -> Instance:
    T, d = 4, 8
    m = m or [20, 18, 16, 14]
    dz = lattice_design(d, m, seed, n_max=1 << m[0])
    Lm = normal(seed, 0x77, np.arange(T * T)).reshape(T, T)
    hp = Hyper(gamma=1.0, eta=0.5 ** np.arange(1, d + 1), B=Lm, t=np.full(T, 0.1), xi=np.full(T, 1e-8),
               si_alpha=2)
    X = uniform01(seed, 0x7E57, np.arange(n_test * d)).reshape(n_test, d)
    return Instance("config3", dz, hp, _y_exp(dz, seed), ("c", "logdet", "posterior_var", "cubature"), X_test=X)


def config4(seed: int = 404, m: Optional[List[int]] = None) -> Instance:
    T, d = 2, 4
    m = m or [26] * T
    dz = lattice_design(d, m, seed)
    w = normal(seed, 0x77, np.arange(T)).reshape(T, 1)
    hp = Hyper(gamma=1.0, eta=np.full(d, 0.8), B=w, t=np.full(T, 0.5), xi=np.full(T, 1e-8), si_alpha=1)
    return Instance("config4", dz, hp, _y_sines(dz, seed), ("nll", "grad"))


def config5(seed: int = 505, m: Optional[List[int]] = None, n_cand: int = 256) -> Instance:
    T, d = 4, 10
    m = m or [18] * T
    dz = digital_design(d, m, seed)
    cands = []
    for c in range(n_cand):
        u = uniform01(seed, 0xE7A + c, np.arange(d))
        eta = np.exp(np.log(1e-2) + u * (np.log(1e1) - np.log(1e-2)))
        Lm = normal(seed, 0x1000 + c, np.arange(T * T)).reshape(T, T)
        cands.append(Hyper(gamma=1.0, eta=eta, B=Lm, t=np.full(T, 0.05), xi=np.full(T, 1e-8),
                           b=(0.0, 0.0, 0.0, 1.0)))
    return Instance("config5", dz, cands[0], _y_prod(dz, seed), ("nll", "grad"), candidates=cands)


CONFIGS = {1: config1, 2: config2, 3: config3, 4: config4, 5: config5}


def make(cfg: int, **kw) -> Instance:
    return CONFIGS[cfg](**kw)
