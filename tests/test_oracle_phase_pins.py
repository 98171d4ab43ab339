"""Pins of the oracle's NEXT(1) functions: pairs of phases generated from their factors,
p = RN(f * t), in radians (the whole method) or in turns (the method from the reduction on,
P:53-54).  Same legend as test_oracle_pins.py: CLOSED, PAPER, SURVEY, LIBM."""
import json
import os

import numpy as np
import pytest

import oracle

R, T = oracle.UNITS_RADIANS, oracle.UNITS_TURNS
VARIANTS = (oracle.VARIANT_N, oracle.VARIANT_A)


def golden_exhaustive():
    p = os.path.join(os.path.dirname(__file__), "golden", "oracle_exhaustive.json")
    return json.load(open(p))


@pytest.mark.parametrize("variant", VARIANTS)
def test_turns_closed_forms(variant):
    """CLOSED: an integral number of turns is (0, 1) exactly; a quarter turn is (1, 0) and a
    half turn (0, -1) to the method's accuracy; x1 = k + 1/2 ties to even (reading G4)."""
    f = np.array([1, 1, 1, 1, 3, 0.25, 0.25, 0.5, 1.5, 2.5, 0.75], dtype=np.float32)
    t = np.array([0, 1, -3, 1e6, 7, 1, -1, 1, 1, 1, 1], dtype=np.float32)
    s, c = oracle.phase_points(f, t, T, variant)
    assert np.all(s[:5] == 0) and np.all(c[:5] == 1)
    assert abs(s[5] - 1) < 5e-7 and abs(c[5]) < 5e-7
    assert abs(s[6] + 1) < 5e-7 and abs(c[6]) < 5e-7
    for k in (7, 8, 9):
        assert abs(c[k] + 1) < 5e-7 and abs(s[k]) < 5e-7
    # 0.5 -> rint 0 -> q = +1/2 ; 1.5 -> rint 2 -> q = -1/2 ; 2.5 -> rint 2 -> q = +1/2
    qp, _ = oracle.pair_from_q(0.5, variant)
    qm, _ = oracle.pair_from_q(-0.5, variant)
    assert s[7] == qp and s[8] == qm and s[9] == qp
    assert abs(s[10] + 1) < 5e-7


@pytest.mark.parametrize("name,variant", [("N", oracle.VARIANT_N), ("A", oracle.VARIANT_A)])
def test_turns_error_within_the_exhaustive_kernel_bound(name, variant):
    """SURVEY [X5] / tests/golden/oracle_exhaustive.json: in turns the only error is the
    kernel's, so against sin/cos(2 pi p) (double) every pair is within the exhaustive
    kernel-only maximum over all q."""
    bound = golden_exhaustive()[name]["q_half"]["max"]
    rng = np.random.default_rng(4)
    f = (512 * rng.random(200000)).astype(np.float32)
    t = rng.random(200000).astype(np.float32)
    s, c = oracle.phase_points(f, t, T, variant)
    p = (f * t).astype(np.float64)                       # fp32 product, exact in double
    p32 = (f * t)                                        # numpy fp32 multiply = RN(f t)
    ref_s, ref_c = np.sin(2 * np.pi * (p32.astype(np.float64) - np.round(p32.astype(np.float64)))), \
        np.cos(2 * np.pi * (p32.astype(np.float64) - np.round(p32.astype(np.float64))))
    err = np.hypot(s - ref_s, c - ref_c)
    assert err.max() <= bound * (1 + 1e-9), err.max()
    assert p.size == s.size


@pytest.mark.parametrize("variant", VARIANTS)
def test_radians_error_model(variant):
    """SURVEY 8(c) G9 (error analysis of the fp32 reduction): for phases in radians the error
    against double sin/cos(p) is at most the kernel term plus 2 pi (|x1| 4.03e-8 + ulp(x1)/2)."""
    rng = np.random.default_rng(5)
    f = (2 * np.pi * 512 * rng.random(200000)).astype(np.float32)
    t = rng.random(200000).astype(np.float32)
    s, c = oracle.phase_points(f, t, R, variant)
    p = (f * t).astype(np.float64)
    err = np.hypot(s - np.sin(p), c - np.cos(p))
    x1 = np.abs(p / (2 * np.pi)).astype(np.float32)
    bound = 4.9e-7 + 2 * np.pi * (x1 * 4.03e-8 + np.spacing(x1) / 2)
    assert np.all(err <= bound * 1.01 + 1e-12)
    # and the radians path equals the theta path on the rounded product (composition)
    th = f * t
    s2, c2 = oracle.sincos(th, variant)
    assert np.array_equal(s, s2) and np.array_equal(c, c2)


def test_turns_are_more_accurate_than_radians_for_large_phases():
    """LIBM (long double via exact products): forming the phase in turns skips the
    1/2pi rounding that dominates large-argument error (SURVEY [X12]); the radians path
    with omega = fl32(2 pi f) loses ~|x1| 2^-24, the turns path stays near the kernel bound."""
    rng = np.random.default_rng(6)
    f = (512 * rng.random(50000)).astype(np.float32)
    t = rng.random(50000).astype(np.float32)
    st, ct = oracle.phase_points(f, t, T, oracle.VARIANT_N)
    om = (2 * np.pi * f.astype(np.float64)).astype(np.float32)
    sr, cr = oracle.phase_points(om, t, R, oracle.VARIANT_N)
    exact = 2 * np.pi * np.fmod(f.astype(np.float64) * t.astype(np.float64), 1.0)
    et = np.hypot(st - np.sin(exact), ct - np.cos(exact)).max()
    er = np.hypot(sr - np.sin(exact), cr - np.cos(exact)).max()
    # turns: one rounding of the product (|p| 2^-24 turns) plus the kernel term
    pmax = float(np.max(np.abs(f.astype(np.float64) * t)))
    assert et <= 2 * np.pi * pmax * 2.0 ** -24 + 4.9e-7
    # radians: the product rounding, the 1/2pi rounding of x1 and K's own error on top
    assert er > 1.8 * et, (er, et)


@pytest.mark.parametrize("units", [R, T])
def test_grid_is_row_major_over_f_then_t(units):
    """CLOSED (layout): element (i, j) of the grid is the pair of f[i] * t[j]."""
    rng = np.random.default_rng(7)
    f = rng.uniform(0, 50, 37).astype(np.float32)
    t = rng.uniform(0, 1, 53).astype(np.float32)
    s, c = oracle.phase_grid(f, t, units, oracle.VARIANT_A)
    ii, jj = np.meshgrid(np.arange(37), np.arange(53), indexing="ij")
    sp_, cp_ = oracle.phase_points(f[ii.ravel()], t[jj.ravel()], units, oracle.VARIANT_A)
    assert np.array_equal(s.ravel(), sp_) and np.array_equal(c.ravel(), cp_)
    assert np.array_equal(s[:, 0], oracle.phase_points(f, np.full(37, t[0], np.float32), units, oracle.VARIANT_A)[0])


def test_bad_arguments():
    with pytest.raises(ValueError):
        oracle.phase_points(np.ones(2), np.ones(2), 2, 0)
    with pytest.raises(ValueError):
        oracle.phase_points(np.ones(2), np.ones(2), 0, 9)
