"""Pin the CPU oracle (our C restatement `oracle.port`, and the reference library itself
`oracle.ref`) against the reference's own known-answer tests, restated here with their
tolerances (SURVEY.md §8c "Golden vectors / KATs to restate")."""
import math

import numpy as np
import pytest

from paper_2603_16014_b200 import designs

PI2 = 9.869604401089358618834491
PI4 = PI2 * PI2

# tests/test_kernels.cpp:62-81 — DSI frozen rational spot values (u, k1..k4)
DSI_TABLE = [
    (0.0, 1.0, 3.0 / 2.0, 25.0 / 18.0, 407.0 / 294.0),
    (0.5, -0.5, -1.0 / 4.0, -5.0 / 24.0, -23.0 / 112.0),
    (0.25, 0.25, 3.0 / 8.0, 41.0 / 96.0, 1157.0 / 2688.0),
    (0.375, 0.25, 1.0 / 8.0, 11.0 / 96.0, 101.0 / 896.0),
    (0.6875, -0.5, -7.0 / 16.0, -349.0 / 768.0, -13035.0 / 28672.0),
]


@pytest.fixture(params=["port", "ref"])
def orc(request, ref, port):
    return port if request.param == "port" else ref


def close(a, b, eps):  # doctest::Approx(b).epsilon(eps)
    return abs(a - b) <= eps * (1.0 + max(abs(a), abs(b)))


def test_si_pinned_values(orc):  # test_kernels.cpp:27-33
    assert close(orc.si_bernoulli_1d(0.3, 0.3, 1), PI2 / 3.0, 1e-14)
    assert close(orc.si_bernoulli_1d(0.75, 0.25, 1), -PI2 / 6.0, 1e-14)
    assert close(orc.si_bernoulli_1d(0.3, 0.3, 2), PI4 / 45.0, 1e-14)
    assert close(orc.si_bernoulli_1d(0.75, 0.25, 2), -7.0 * PI4 / 360.0, 1e-14)


def test_si_zero_mean_and_symmetry(orc):  # test_kernels.cpp:35-48
    n = 1 << 12
    for alpha in (1, 2):
        mean = sum(orc.si_bernoulli_1d((k + 0.5) / n, 0.0, alpha) for k in range(n)) / n
        assert abs(mean) < 1e-6
    u = designs.uniform01(31, 0, np.arange(100))
    for k in range(50):
        x, y = float(u[2 * k]), float(u[2 * k + 1])
        assert orc.si_bernoulli_1d(x, y, 1) == orc.si_bernoulli_1d(y, x, 1)
        assert orc.si_bernoulli_1d(x, y, 2) == orc.si_bernoulli_1d(y, x, 2)


@pytest.mark.parametrize("row", DSI_TABLE)
def test_dsi_rational_table(orc, row):  # test_kernels.cpp:62-81
    u = row[0]
    for alpha in range(1, 5):
        assert close(orc.dsi_order_1d(alpha, u, 0.0), row[alpha], 1e-14)


def test_dsi_shift_invariance(orc):  # test_kernels.cpp:93-102
    b = designs.bits53(33, 0, np.arange(300))
    for k in range(100):
        x, y, s = (int(v) for v in b[3 * k:3 * k + 3])
        xs, ys = designs.bits_to_frac(np.uint64(x ^ s)), designs.bits_to_frac(np.uint64(y ^ s))
        for alpha in range(1, 5):
            assert orc.dsi_order_1d(alpha, float(xs), float(ys)) == orc.dsi_order_1d(
                alpha, float(designs.bits_to_frac(np.uint64(x))), float(designs.bits_to_frac(np.uint64(y))))


def test_fwht_pins_and_involution(orc):  # test_transforms.cpp:54-77
    a = orc.fwht([1.0, 1.0])
    assert close(a[0], math.sqrt(2.0), 1e-15) and abs(a[1]) <= 1e-15
    e = orc.fwht([1.0, 0.0, 0.0, 0.0])
    assert all(close(v, 0.5, 1e-15) for v in e)
    x = designs.normal(7, 1, np.arange(64))
    y = orc.fwht(orc.fwht(x))
    assert np.allclose(y, x, rtol=1e-12, atol=1e-12)
    assert close(float(np.sum(orc.fwht(x) ** 2)), float(np.sum(x ** 2)), 1e-12)


def _dft(a, sign):
    n = len(a)
    j = np.arange(n)
    return np.exp(sign * 2j * np.pi * np.outer(j, j) / n) @ a / math.sqrt(n)


def test_fft_bitrev_conventions(orc):  # test_transforms.cpp:79-140
    n, m = 16, 4
    a = designs.normal(13, 2, np.arange(2 * n))[0::2] + 1j * designs.normal(13, 2, np.arange(2 * n))[1::2]
    perm = np.empty(n, dtype=complex)
    perm[designs.bit_reverse(np.arange(n), m).astype(int)] = a
    assert np.linalg.norm(orc.fft_bitrev(a) - _dft(perm, -1)) < 1e-12
    want = np.empty(n, dtype=complex)
    want[designs.bit_reverse(np.arange(n), m).astype(int)] = _dft(a, +1)
    assert np.linalg.norm(orc.fft_bitrev(a, inverse=True) - want) < 1e-12
    for nn in (1, 4, 32, 256):
        v = designs.normal(4, nn, np.arange(nn)) + 0j
        w = orc.fft_bitrev(v)
        assert close(float(np.vdot(w, w).real), float(np.vdot(v, v).real), 1e-12)
        assert np.linalg.norm(orc.fft_bitrev(w, inverse=True) - v) < 1e-11
    c = np.full(8, 2.0 + 1.0j)
    w = orc.fft_bitrev(c)
    assert abs(w[0] - c[0] * math.sqrt(8)) < 1e-13 and np.all(np.abs(w[1:]) < 1e-13)
    r = orc.fft_bitrev(designs.normal(21, 5, np.arange(32)) + 0j)
    assert abs(r[0].imag) < 1e-13
    assert np.all(np.abs(r[1:] - np.conj(r[1:][::-1])) < 1e-12)


def test_lattice_points_small_generator(ref, port):  # test_rng_sequences.cpp:50-66
    dz = designs.Design(designs.LATTICE, 2, [2], np.zeros((1, 2), np.uint64), g=np.array([1, 3], np.uint64),
                        n_max=1 << 20)
    for orc in (ref, port):
        pts = orc.design_points(dz)
        assert list(pts[0]) == [0.0, 0.0] and list(pts[1]) == [0.5, 0.5]
        assert list(pts[2]) == [0.25, 0.75] and list(pts[3]) == [0.75, 0.25]
    assert np.array_equal(designs.bits_to_frac(dz.point_bits(0)), ref.design_points(dz))


def test_rng_matches_reference(ref, port):  # rng.hpp:14-47
    for s, st, c in [(1, 2, 3), (9, 0, 17), (2 ** 63, 5, 2 ** 40)]:
        want = ref.lib().ref_rand_u64(s, st, c)
        assert int(designs.rand_u64(s, st, np.array([c]))[0]) == want
        assert port.lib().orc_rand_u64(s, st, c) == want
        assert port.lib().orc_normal(s, st, c) == ref.lib().ref_normal(s, st, c)
