"""The seeded input generators (inputs/): determinism, ranges and the shape of each config's
distribution."""
import math

import numpy as np

import inputs


def test_sizes():
    assert [inputs.size(c) for c in (1, 2, 3, 4, 5)] == [1 << 20, 1 << 28, 1 << 24, 1 << 30, 1 << 32]


def test_urand_is_counter_based_uniform():
    u = np.array([inputs.urand(9, 0, i) for i in range(20000)])
    assert u.min() >= 0 and u.max() < 1
    assert abs(u.mean() - 0.5) < 0.01 and abs(u.var() - 1 / 12) < 0.005
    assert inputs.urand(9, 0, 5) == inputs.urand(9, 0, 5) != inputs.urand(9, 1, 5)


def test_ranges_and_samples_agree_and_do_not_depend_on_threads():
    for c in (1, 2, 3, 4, 5):
        a = inputs.generate(c, 1000, 5000, nthreads=1)
        b = inputs.generate(c, 1000, 5000, nthreads=4)
        assert np.array_equal(a.view(np.uint32), b.view(np.uint32))
        idx = np.array([1000, 1001, 5999, 3333], dtype=np.uint64)
        assert np.array_equal(inputs.generate_at(c, idx).view(np.uint32), a[(idx - 1000).astype(np.int64)].view(np.uint32))


def test_c1_c2_uniform_ranges():
    a = inputs.generate(1)
    assert a.size == 1 << 20 and a.min() >= -np.float32(math.pi) and a.max() <= np.float32(math.pi)
    assert abs(a.mean()) < 0.01
    b = inputs.generate(2, 0, 1 << 20)
    assert b.min() >= -1e4 and b.max() <= 1e4 and abs(b.mean()) < 30


def test_c3_categories():
    a = inputs.generate(3, 0, 1 << 18).astype(np.float64)
    absa = np.abs(a)
    # signed zeros ~ 1/16, subnormals ~ 2/16
    assert abs(np.mean(a == 0) - 1 / 16) < 0.005
    sub = (absa > 0) & (absa < 2.0 ** -126)
    assert abs(np.mean(sub) - 2 / 16) < 0.005
    # near-wrap values: within 64 ulp of an odd multiple of pi, ~4/16
    m = np.round(absa / math.pi)
    near_wrap = (m % 2 == 1) & (np.abs(absa - m * math.pi) < 64 * np.spacing(absa.astype(np.float32)) + 1e-6) & (absa >= 3)
    assert np.mean(near_wrap) > 3.5 / 16
    assert absa.max() <= 2.0 ** 20
    assert np.any(np.signbit(a[a == 0])) and np.any(~np.signbit(a[a == 0]))


def test_c4_phase_structure():
    row = inputs.generate(4, 5 << 15, 1 << 15).astype(np.float64)
    assert np.all(np.diff(row) >= 0)                     # t_j sorted, f_i >= 0
    t = np.array([(j + inputs.urand(3, 1, j)) * 2.0 ** -15 for j in range(1 << 15)])
    f = 512 * inputs.urand(3, 0, 5)
    np.testing.assert_allclose(row, (2 * math.pi * f) * t, rtol=1e-7)
    assert np.all(np.diff(t) > 0) and np.diff(t).max() < 2.0 ** -14   # non-uniform spacing in (0, 2^-14)


def test_c5_normal():
    a = inputs.generate(5, 0, 1 << 20).astype(np.float64)
    assert abs(a.mean()) < 0.5 and abs(a.std() - 100) < 0.5
