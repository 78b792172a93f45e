"""Seeded inputs: designs match the reference's point construction exactly, and the
generators have the group structure the fast algorithm needs (test_rng_sequences.cpp)."""
import numpy as np
import pytest

from paper_2603_16014_b200 import configs, designs


@pytest.mark.parametrize("kind", [designs.LATTICE, designs.DIGITAL])
def test_points_bit_identical_to_reference(ref, kind):
    dz = (designs.lattice_design if kind == designs.LATTICE else designs.digital_design)(3, [6, 4, 4], seed=5)
    assert np.array_equal(dz.all_points(), ref.design_points(dz))


def test_lattice_group_closure():  # test_rng_sequences.cpp:112-129
    dz = designs.lattice_design(3, [4], seed=1)
    dz.shift_bits[:] = 0
    pts = {tuple(p) for p in dz.point_bits(0).tolist()}
    mask = (1 << 53) - 1
    for a in pts:
        for b in pts:
            assert tuple((x + y) & mask for x, y in zip(a, b)) in pts


def test_digital_net_group_closure_and_distinct():  # test_rng_sequences.cpp:131-145
    dz = designs.digital_design(4, [6], seed=2)
    dz.shift_bits[:] = 0
    pts = [tuple(p) for p in dz.point_bits(0).tolist()]
    assert len(set(pts)) == 64  # scrambled generator stays non-singular
    s = set(pts)
    for a in pts[:16]:
        for b in pts:
            assert tuple(x ^ y for x, y in zip(a, b)) in s


def test_sobol_first_dimension_is_van_der_corput():  # test_rng_sequences.cpp:41-48, 86-91
    cols = designs.sobol_type_columns(3, 10, seed=3)
    for p in range(10):
        assert designs.bits_to_frac(cols[0, p]) == 2.0 ** -(p + 1)
    pp = designs.primitive_polynomials(6)
    assert pp == [3, 7, 11, 13, 19, 25]


def test_extensible_prefixes():  # test_rng_sequences.cpp:102-110
    for mk in (designs.lattice_design, designs.digital_design):
        dz = mk(3, [7], seed=11)
        a = dz.point_bits(0, 0, 8)
        b = dz.point_bits(0, 0, 32)
        assert np.array_equal(a, b[:8])
        assert np.array_equal(dz.point_bits(0, 8, 24), b[8:])


def test_configs_shapes():
    c1 = configs.make(1)
    assert c1.design.N == 2048 and c1.X_test.shape == (4096, 2)
    c3 = configs.make(3, m=[8, 6, 4, 2], n_test=16)
    assert c3.design.m == [8, 6, 4, 2] and c3.design.n_max == 256
    c5 = configs.make(5, m=[4] * 4, n_cand=8)
    assert len(c5.candidates) == 8
    etas = np.array([h.eta for h in c5.candidates])
    assert etas.min() >= 1e-2 and etas.max() <= 1e1
    assert np.all(np.linalg.eigvalsh(c5.candidates[0].R) > 0)
