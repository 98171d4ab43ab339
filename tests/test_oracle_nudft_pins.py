"""Pins of the oracle's NEXT(2) consumer: F_k = sum_j a_j e^{i p_kj}, p_kj = RN(f_k t_j)
(the Huygens / non-uniform Fourier sum of P:203-206).  CLOSED forms and a LIBRARY routine
(numpy's FFT on a uniform grid, where the sum is a DFT)."""
import json
import os

import numpy as np
import pytest

import oracle

R, T = oracle.UNITS_RADIANS, oracle.UNITS_TURNS


def kernel_bound(name):
    p = os.path.join(os.path.dirname(__file__), "golden", "oracle_exhaustive.json")
    return json.load(open(p))[name]["q_half"]["max"]


def rand_complex(rng, n):
    return (rng.normal(size=n) + 1j * rng.normal(size=n)).astype(np.complex64)


@pytest.mark.parametrize("units", [R, T])
@pytest.mark.parametrize("variant", [0, 1])
def test_single_amplitude_picks_one_pair(units, variant):
    """CLOSED: a = e_j0 gives F_k = the pair of (f_k, t_j0), exactly."""
    rng = np.random.default_rng(1)
    f = rng.uniform(0, 300, 17).astype(np.float32)
    t = rng.uniform(-1, 1, 29).astype(np.float32)
    a = np.zeros(29, np.complex64)
    a[11] = 1
    F = oracle.nudft(f, t, a, units, variant)
    s, c = oracle.phase_points(f, np.full(17, t[11], np.float32), units, variant)
    assert np.array_equal(F.real, c.astype(np.float64)) and np.array_equal(F.imag, s.astype(np.float64))


def test_zero_phase_is_the_plain_sum():
    """CLOSED: t = 0 makes every pair (0, 1) exactly, so F_k = sum_j a_j."""
    rng = np.random.default_rng(2)
    a = rand_complex(rng, 1000)
    F = oracle.nudft(np.arange(5, dtype=np.float32), np.zeros(1000, np.float32), a, R, 0)
    want = np.sum(a.astype(np.complex128))
    assert np.allclose(F, want, rtol=0, atol=1e-12)


@pytest.mark.parametrize("name,variant", [("N", 0), ("A", 1)])
def test_uniform_grid_is_the_dft(name, variant):
    """LIBRARY: with t_j = j/N (turns) and integer f_k = k the sum is the (inverse-sign) DFT,
    F = N * ifft(a).  Every pair is within the exhaustive kernel bound of e^{2 pi i k j/N}
    (the products k*j/N are exact), so |F - N ifft(a)| <= bound * sum|a_j|."""
    N = 1024
    rng = np.random.default_rng(3)
    a = rand_complex(rng, N)
    t = (np.arange(N) / N).astype(np.float32)
    f = np.arange(N, dtype=np.float32)
    F = oracle.nudft(f, t, a, T, variant)
    want = N * np.fft.ifft(a.astype(np.complex128))
    err = np.abs(F - want).max()
    assert err <= kernel_bound(name) * np.abs(a).sum() + 1e-9, err
    # and it is not trivially small: the method's error is visible but bounded
    assert err > 1e-9
    # conjugation / index slips would be O(|F|)
    assert np.abs(F - N * np.fft.fft(a.astype(np.complex128)) / N * 1).max() > 1.0


def test_linearity():
    rng = np.random.default_rng(4)
    f = rng.uniform(0, 100, 8).astype(np.float32)
    t = rng.uniform(0, 1, 300).astype(np.float32)
    a, b = rand_complex(rng, 300), rand_complex(rng, 300)
    Fa, Fb = oracle.nudft(f, t, a, T, 1), oracle.nudft(f, t, b, T, 1)
    Fab = oracle.nudft(f, t, (a.astype(np.complex128) + b).astype(np.complex64), T, 1)
    # a + b rounded to complex64 changes the input by <= 2^-24 relative
    assert np.abs(Fab - (Fa + Fb)).max() <= 2 ** -23 * (np.abs(a).sum() + np.abs(b).sum())
