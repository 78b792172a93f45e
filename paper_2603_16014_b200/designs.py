"""Seeded inputs shared by the GPU path, the oracle and the benchmarks.

Host-side plumbing (numpy), not a GPU kernel.  Every array handed to the CUDA
library and to the CPU oracle comes from here, so both sides see identical bits.

* ``rand_u64 / bits53 / uniform01 / normal`` restate the reference counter RNG
  (nested splitmix64), ``/root/reference/proj/include/fastmtgp/rng.hpp:14-47``.
* ``Design`` mirrors the public aggregate ``LdDesign``
  (``ld_sequences.hpp:56-77``) in internal (descending-n) order; points are
  53-bit fixed-point integers exactly as ``lattice_points`` /
  ``digital_net_points`` produce them (``ld_sequences.cpp:31-87``).
* Generators the reference cannot make: seeded odd lattice
  vectors with any n_max, and Sobol'-type digital nets (primitive polynomials +
  seeded odd initial direction numbers) with seeded linear-matrix scrambling.
"""
from __future__ import annotations

import dataclasses
import math
from typing import List, Optional

import numpy as np

MASK64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15
DIGITAL_BITS = 53
MASK53 = (1 << DIGITAL_BITS) - 1

# --------------------------------------------------------------------------------------
# counter RNG (rng.hpp:14-47)
# --------------------------------------------------------------------------------------


def _mix64(z: np.ndarray) -> np.ndarray:
    z = z ^ (z >> np.uint64(30))
    z = z * np.uint64(0xBF58476D1CE4E5B9)
    z = z ^ (z >> np.uint64(27))
    z = z * np.uint64(0x94D049BB133111EB)
    z = z ^ (z >> np.uint64(31))
    return z


def rand_u64(seed: int, stream: int, counter) -> np.ndarray:
    """rng.hpp:23-29 — vectorised over ``counter``."""
    with np.errstate(over="ignore"):
        sub = _mix64(np.array([(seed + GOLDEN * (stream + 1)) & MASK64], dtype=np.uint64))[0]
        c = np.asarray(counter, dtype=np.uint64)
        return _mix64(sub + np.uint64(GOLDEN) * (c + np.uint64(1)))


def bits53(seed: int, stream: int, counter) -> np.ndarray:
    return rand_u64(seed, stream, counter) >> np.uint64(11)


def uniform01(seed: int, stream: int, counter) -> np.ndarray:
    return bits53(seed, stream, counter).astype(np.float64) * 2.0 ** -53


def normal(seed: int, stream: int, k) -> np.ndarray:
    """Box-Muller on counters 2k, 2k+1 (rng.hpp:42-47)."""
    k = np.asarray(k, dtype=np.uint64)
    u1 = uniform01(seed, stream, k * np.uint64(2))
    u2 = uniform01(seed, stream, k * np.uint64(2) + np.uint64(1))
    u1 = np.where(u1 <= 0.0, 2.0 ** -53, u1)
    return np.sqrt(-2.0 * np.log(u1)) * np.cos(6.283185307179586476925287 * u2)


# --------------------------------------------------------------------------------------
# bit helpers
# --------------------------------------------------------------------------------------


def bit_reverse(i: np.ndarray, m: int) -> np.ndarray:
    """transforms.cpp:10-17, vectorised."""
    i = np.asarray(i, dtype=np.uint64)
    r = np.zeros_like(i)
    for _ in range(m):
        r = (r << np.uint64(1)) | (i & np.uint64(1))
        i = i >> np.uint64(1)
    return r


def bits_to_frac(b: np.ndarray) -> np.ndarray:
    return np.asarray(b, dtype=np.uint64).astype(np.float64) * 2.0 ** -53


# --------------------------------------------------------------------------------------
# designs
# --------------------------------------------------------------------------------------

LATTICE = 0
DIGITAL = 1


@dataclasses.dataclass
class Design:
    """Per-task shifted point sets sharing one generator (internal order)."""

    kind: int  # LATTICE | DIGITAL
    d: int
    m: List[int]  # descending log2 sizes
    shift_bits: np.ndarray  # [L, d] uint64, 53-bit fractions
    g: Optional[np.ndarray] = None  # lattice [d] uint64, g[0] == 1
    n_max: int = 0  # lattice
    columns: Optional[np.ndarray] = None  # digital [d, m_cols] uint64 (53-bit msb-aligned)

    def __post_init__(self):
        self.shift_bits = np.ascontiguousarray(self.shift_bits, dtype=np.uint64).reshape(self.L, self.d)
        if any(self.m[i] < self.m[i + 1] for i in range(self.L - 1)):
            raise ValueError("Design: task sizes must be descending (internal order)")
        if self.kind == LATTICE:
            self.g = np.ascontiguousarray(self.g, dtype=np.uint64)
            if self.n_max < (1 << self.m[0]):
                raise ValueError("Design: n_max below the largest task size")
        else:
            self.columns = np.ascontiguousarray(self.columns, dtype=np.uint64)
            if self.columns.shape[1] < self.m[0]:
                raise ValueError("Design: not enough digital columns for the largest task")

    @property
    def L(self) -> int:
        return len(self.m)

    @property
    def n(self) -> List[int]:
        return [1 << mm for mm in self.m]

    @property
    def offset(self) -> List[int]:
        o = [0]
        for nn in self.n:
            o.append(o[-1] + nn)
        return o

    @property
    def N(self) -> int:
        return sum(self.n)

    @property
    def m_cols(self) -> int:
        return 0 if self.columns is None else int(self.columns.shape[1])

    def point_bits(self, l: int, i0: int = 0, count: Optional[int] = None) -> np.ndarray:
        """[count, d] uint64 point bits of task l (ld_sequences.cpp:31-53 / 64-87)."""
        if count is None:
            count = (1 << self.m[l]) - i0
        idx = np.arange(i0, i0 + count, dtype=np.uint64)
        out = np.empty((count, self.d), dtype=np.uint64)
        if self.kind == LATTICE:
            mgen = int(round(math.log2(self.n_max)))
            k = bit_reverse(idx, mgen)
            mask = np.uint64(self.n_max - 1)
            with np.errstate(over="ignore"):
                for j in range(self.d):
                    frac = ((k * self.g[j]) & mask) << np.uint64(DIGITAL_BITS - mgen)
                    out[:, j] = (frac + self.shift_bits[l, j]) & np.uint64(MASK53)
        else:
            for j in range(self.d):
                z = np.full(count, self.shift_bits[l, j], dtype=np.uint64)
                for p in range(max(1, int(i0 + count - 1).bit_length())):
                    sel = ((idx >> np.uint64(p)) & np.uint64(1)).astype(bool)
                    z[sel] ^= self.columns[j, p]
                out[:, j] = z
        return out

    def points(self, l: int) -> np.ndarray:
        return bits_to_frac(self.point_bits(l))

    def all_points(self) -> np.ndarray:
        return np.concatenate([self.points(l) for l in range(self.L)], axis=0)


def lattice_generator(d: int, n_max: int, seed: int, stream: int = 0x1A7) -> np.ndarray:
    """Seeded odd generating vector in [1, n_max), first component 1 (BASELINE configs)."""
    u = uniform01(seed, stream, np.arange(d))
    g = 2 * np.floor(u * (n_max // 2)).astype(np.uint64) + np.uint64(1)
    g[0] = 1
    return g


def _gf2_mulmod(a: int, b: int, p: int, deg: int) -> int:
    r = 0
    while b:
        if b & 1:
            r ^= a
        b >>= 1
        a <<= 1
        if a >> deg & 1:
            a ^= p
    return r


def _gf2_powmod(a: int, e: int, p: int, deg: int) -> int:
    r = 1
    while e:
        if e & 1:
            r = _gf2_mulmod(r, a, p, deg)
        a = _gf2_mulmod(a, a, p, deg)
        e >>= 1
    return r


def _prime_factors(x: int) -> List[int]:
    out, q = [], 2
    while q * q <= x:
        if x % q == 0:
            out.append(q)
            while x % q == 0:
                x //= q
        q += 1
    if x > 1:
        out.append(x)
    return out


def primitive_polynomials(count: int) -> List[int]:
    """First ``count`` primitive polynomials over GF(2), by degree (bit s = x^s)."""
    found: List[int] = []
    deg = 1
    while len(found) < count:
        order = (1 << deg) - 1
        for p in range(1 << deg, 1 << (deg + 1)):
            if not p & 1:
                continue
            if deg == 1:
                ok = True
            else:
                ok = _gf2_powmod(2, order, p, deg) == 1 and all(
                    _gf2_powmod(2, order // q, p, deg) != 1 for q in _prime_factors(order)
                )
            if ok:
                found.append(p)
                if len(found) == count:
                    break
        deg += 1
    return found


def sobol_type_columns(d: int, m_cols: int, seed: int, stream: int = 0x50B) -> np.ndarray:
    """Sobol' direction numbers, 53-bit msb-aligned: dim 0 is van der Corput; dim j>=1
    uses the j-th primitive polynomial with seeded odd initial m_k < 2^k."""
    cols = np.zeros((d, m_cols), dtype=np.uint64)
    polys = primitive_polynomials(max(d - 1, 1))
    ctr = 0
    for j in range(d):
        mvals: List[int] = []
        if j == 0:
            mvals = [1] * m_cols
        else:
            p = polys[j - 1]
            s = p.bit_length() - 1
            for k in range(1, s + 1):
                u = float(uniform01(seed, stream, ctr))
                ctr += 1
                mvals.append(2 * int(u * (1 << (k - 1))) + 1)  # odd, < 2^k
            for k in range(s + 1, m_cols + 1):
                v = mvals[k - s - 1] ^ (mvals[k - s - 1] << s)
                for i in range(1, s):
                    if p >> (s - i) & 1:
                        v ^= mvals[k - i - 1] << i
                mvals.append(v)
            mvals = mvals[:m_cols]
        for p_ in range(m_cols):
            cols[j, p_] = np.uint64(mvals[p_] << (DIGITAL_BITS - (p_ + 1)))
    return cols


def lms_scramble(cols: np.ndarray, seed: int, stream: int = 0x135) -> np.ndarray:
    """Left-multiply each dimension's generator by a seeded random unit lower-triangular
    53x53 binary matrix (digit 1 = msb)."""
    d, mc = cols.shape
    out = np.zeros_like(cols)
    ctr = 0
    for j in range(d):
        rows = []
        for r in range(DIGITAL_BITS):
            rnd = int(bits53(seed, stream, np.array([ctr]))[0])
            ctr += 1
            pos = DIGITAL_BITS - 1 - r
            mask = ((rnd >> (pos + 1)) << (pos + 1)) & MASK53  # digits above r (more significant)
            rows.append(mask | (1 << pos))
        for p in range(mc):
            c = int(cols[j, p])
            v = 0
            for r in range(DIGITAL_BITS):
                if bin(c & rows[r]).count("1") & 1:
                    v |= 1 << (DIGITAL_BITS - 1 - r)
            out[j, p] = np.uint64(v)
    return out


def lattice_design(d: int, m: List[int], seed: int, n_max: Optional[int] = None) -> Design:
    n_max = n_max or (1 << m[0])
    shifts = np.stack([bits53(seed, 0x5A1 + l, np.arange(d)) for l in range(len(m))])
    return Design(LATTICE, d, list(m), shifts, g=lattice_generator(d, n_max, seed), n_max=n_max)


def digital_design(d: int, m: List[int], seed: int, m_cols: int = 32, scramble: bool = True) -> Design:
    cols = sobol_type_columns(d, m_cols, seed)
    if scramble:
        cols = lms_scramble(cols, seed)
    shifts = np.stack([bits53(seed, 0xD15 + l, np.arange(d)) for l in range(len(m))])
    return Design(DIGITAL, d, list(m), shifts, columns=cols)


# --------------------------------------------------------------------------------------
# hyperparameters (kernels.hpp:21-31 Hyperparams; task_gram kernels.cpp:124-135)
# --------------------------------------------------------------------------------------


@dataclasses.dataclass
class Hyper:
    gamma: float
    eta: np.ndarray  # [d]
    B: np.ndarray  # [L, s]  (BASELINE w / L)
    t: np.ndarray  # [L]     (BASELINE v)
    xi: np.ndarray  # [L]
    si_alpha: int = 1  # 1 -> B2, 2 -> B4 (lattice)
    b: tuple = (0.0, 0.0, 0.0, 1.0)  # DSI order weights (digital); order-4 Walsh = e4

    def __post_init__(self):
        self.eta = np.ascontiguousarray(self.eta, dtype=np.float64)
        self.B = np.ascontiguousarray(np.atleast_2d(self.B), dtype=np.float64)
        self.t = np.ascontiguousarray(self.t, dtype=np.float64)
        self.xi = np.ascontiguousarray(self.xi, dtype=np.float64)

    @property
    def R(self) -> np.ndarray:
        if np.any(~(self.t > 0)):
            raise ValueError("task_gram: non-positive diagonal entry")
        return self.B @ self.B.T + np.diag(self.t)

    def replace(self, **kw) -> "Hyper":
        return dataclasses.replace(self, **kw)
