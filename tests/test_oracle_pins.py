"""Pins of the ORACLE to things other than itself (CPU only, ``-m "not gpu"``).

Each test names what fixes the expected value:
  PAPER   a value or statement printed in PAPER.md (line cited; tests/golden/paper_values.json)
  CLOSED  a closed form / special case of the mathematics
  LIBM    double libm or long-double sinl/cosl (the paper's own reference)
  SURVEY  the survey author's independent C transcription (SURVEY.md App. A,
          tests/golden/survey_crosscheck.json) -- catches transcription slips
          (a dropped FMA, the wrong fix pair, the wrong ss2) bit for bit
  EXACT   exact rational arithmetic with explicit IEEE rounding (catches
          compiler contraction / excess precision in the C build)
DESIGN.md "Oracle and its pins" maps each plausible mistake to the test that
catches it.
"""
import math
import struct
from fractions import Fraction

import numpy as np
import pytest

import oracle


def f32(x) -> np.float32:
    return np.float32(x)


def bits(x) -> int:
    return struct.unpack("<I", struct.pack("<f", float(x)))[0]


def from_bits(u: int) -> float:
    return struct.unpack("<f", struct.pack("<I", u & 0xFFFFFFFF))[0]


def fl32_pi():
    return float(np.float32(math.pi))


def paper_coeffs(golden, name):
    c = golden["paper_values"]["coefficients"][name]
    return [Fraction(s) for s in c["ss"]], [Fraction(s) for s in c["cc"]]


# --------------------------------------------------------------------------
# constants and coefficients
# --------------------------------------------------------------------------

def test_coefficients_are_the_papers_digits(golden):
    """PAPER P:140-148, Fig. 1 P:228-258 (+ SURVEY [X1] hex table)."""
    hexes = golden["survey_crosscheck"]["constants_hex"]
    for name, variant in (("N", oracle.VARIANT_N), ("A", oracle.VARIANT_A)):
        k = oracle.opts(variant).coeffs
        ss, cc = golden["paper_values"]["coefficients"][name]["ss"], golden["paper_values"]["coefficients"][name]["cc"]
        got = [k.ss1, k.ss2, k.ss3, k.ss4, k.cc1, k.cc2, k.cc3]
        want = [float(np.float32(float(s))) for s in ss + cc]
        assert got == want, name
        for fld, g in zip(("ss1", "ss2", "ss3", "ss4", "cc1", "cc2", "cc3"), got):
            assert bits(g) == int(hexes[name][fld], 16), (name, fld)
    kt = oracle.opts(oracle.VARIANT_A_TEXT).coeffs
    assert bits(kt.ss2) == int(hexes["A_text_ss2"], 16)
    # the text and Fig. 1 values of ss2 are one ulp apart (reading G1)
    assert bits(kt.ss2) - bits(oracle.opts(oracle.VARIANT_A).coeffs.ss2) == 1


def test_signs_alternate_and_ss1_is_half_pi(golden):
    """CLOSED: sin(pi x/2) = (pi/2) x - ..., cos(pi x/2) = 1 - (pi^2/8) x^2 + ... (Taylor)."""
    for v in (oracle.VARIANT_N, oracle.VARIANT_A):
        k = oracle.opts(v).coeffs
        assert k.ss1 > 0 > k.ss2 and k.ss3 > 0 > k.ss4
        assert k.cc1 < 0 < k.cc2 and k.cc3 < 0
        assert abs(k.ss1 - math.pi / 2) < 2e-7
        assert abs(k.cc1 + math.pi ** 2 / 8) < 2e-3      # LS/angle fits perturb the Taylor value
        assert abs(k.ss2 + math.pi ** 3 / 48) < 2e-3


# --------------------------------------------------------------------------
# A1 turn reduction (Fig. 1)
# --------------------------------------------------------------------------

def test_scale_constant_is_fl32_inverse_two_pi(golden):
    """PAPER P:270 constant 1/(2*3.1415926536) == fl32(1/(2 pi)) (reading G12; SURVEY [X1])."""
    k = np.float32(eval(golden["paper_values"]["scale_constant"]["expr"]))
    assert bits(k) == int(golden["survey_crosscheck"]["constants_hex"]["K"], 16)
    assert k == np.float32(1 / (2 * math.pi))
    # the oracle uses it: theta = 1/K maps to x1 = RN(1/K * K), within an ulp of one turn
    assert oracle.reduce_turns(0.0) == 0.0


def test_reduce_turns_closed_forms():
    """CLOSED: q = x1 - round_half_even(x1) at exactly representable turns."""
    assert oracle.reduce_turns(0.0) == 0.0
    assert oracle.reduce_turns(float(np.float32(math.pi / 2))) == 0.25      # SURVEY [X7]
    assert oracle.reduce_turns(fl32_pi()) == 0.5
    assert oracle.reduce_turns(-fl32_pi()) == -0.5
    assert oracle.reduce_turns(2.0 ** 30) == 0.0           # |x1| >= 2^23: integral, q = 0
    assert oracle.reduce_turns(3.0e38) == 0.0
    assert math.isnan(oracle.reduce_turns(float("nan")))
    assert math.isnan(oracle.reduce_turns(float("inf")))    # Inf - Inf
    assert math.isnan(oracle.reduce_turns(float("-inf")))


def _theta_with_x1(x1: float) -> float:
    """An fp32 theta whose fp32 product theta*K is exactly x1 (input search only)."""
    k = np.float32(1 / (2 * math.pi))
    t0 = np.float32(x1 * 2 * math.pi)
    u0 = bits(t0)
    for d in range(-64, 65):
        t = np.float32(from_bits(u0 + d))
        if np.float32(t * k) == np.float32(x1):
            return float(t)
    raise AssertionError("no partner")


@pytest.mark.parametrize("x1,q", [(1.5, -0.5), (2.5, 0.5), (-1.5, 0.5), (-2.5, -0.5), (0.5, 0.5), (14.5, 0.5)])
def test_reduce_turns_ties_to_even(x1, q):
    """CLOSED + reading G4 (vec_round = nearest, ties to even): x1 = 2.5 -> round 2 -> q=+0.5
    (round-half-away would give 3 -> q=-0.5)."""
    theta = _theta_with_x1(x1)
    assert oracle.reduce_turns(theta) == q
    if x1 == 1.5:
        assert bits(theta) == 0x4116CBE4     # SURVEY [X7]


def test_reduce_turns_range_and_exactness():
    """CLOSED: q in [-1/2, 1/2] and q + round(x1) == x1 exactly."""
    rng = np.random.default_rng(1)
    th = np.concatenate([rng.uniform(-1e4, 1e4, 2000), rng.uniform(-10, 10, 2000),
                         np.float32(10.0) ** rng.uniform(-30, 30, 2000)]).astype(np.float32)
    k = Fraction(float(np.float32(1 / (2 * math.pi))))
    for t in th[:3000]:
        q = oracle.reduce_turns(float(t))
        assert -0.5 <= q <= 0.5
        x1 = rn32(Fraction(float(t)) * k)
        assert Fraction(q) == x1 - round(x1)


# --------------------------------------------------------------------------
# exact rational emulation (EXACT)
# --------------------------------------------------------------------------

def rn32(x: Fraction) -> Fraction:
    """Round an exact rational to the nearest fp32, ties to even (IEEE RN)."""
    f = np.float32(float(x))
    cands = [np.nextafter(f, np.float32(-np.inf)), f, np.nextafter(f, np.float32(np.inf))]
    best, bd = None, None
    for c in cands:
        if not np.isfinite(c):
            continue
        d = abs(Fraction(float(c)) - x)
        if bd is None or d < bd or (d == bd and (bits(c) & 1) == 0):
            best, bd = c, d
    return Fraction(float(best))


def fma(a, b, c):
    return rn32(Fraction(a) * Fraction(b) + Fraction(c))


def exact_pipeline(theta: float, variant: int):
    """Fig. 1 P:270-360 in exact rationals with one IEEE rounding per AltiVec op."""
    o = oracle.opts(variant)
    k = o.coeffs
    K = Fraction(float(np.float32(1.0 / (2.0 * 3.1415926536))))
    x1 = fma(theta, K, 0)
    q1 = fma(-round(x1), 1, x1)
    q2 = fma(q1, q1, 0)
    s1 = fma(q1, fma(q2, fma(q2, fma(q2, k.ss4, k.ss3), k.ss2), k.ss1), 0)
    c1 = fma(q2, fma(q2, fma(q2, k.cc3, k.cc2), k.cc1), 1)
    c2 = fma(-s1, s1, fma(c1, c1, 0))
    s2 = fma(2, fma(s1, c1, 0), 0)
    if variant == oracle.VARIANT_N:
        fix = fma(-s2, s2, fma(-c2, c2, 2))
    else:
        fix = rn32(1 / fma(s2, s2, fma(c2, c2, 0)))
    c3 = fma(-s2, s2, fma(c2, c2, 0))
    s3 = fma(2, fma(s2, c2, 0), 0)
    return float(fma(s3, fix, 0)), float(fma(c3, fix, 0))


@pytest.mark.parametrize("variant", [oracle.VARIANT_N, oracle.VARIANT_A])
def test_oracle_build_matches_exact_rounding(variant):
    """EXACT: the compiled oracle rounds exactly once per operation (no contraction / x87)."""
    rng = np.random.default_rng(7 + variant)
    th = np.concatenate([rng.uniform(-math.pi, math.pi, 300), rng.uniform(-1e4, 1e4, 200),
                         [0.0, fl32_pi(), -fl32_pi(), float(np.float32(math.pi / 2)), 1e-40,
                          _theta_with_x1(2.5), _theta_with_x1(1.5)]]).astype(np.float32)
    s, c = oracle.sincos(th, variant)
    for t, si, ci in zip(th, s, c):
        es, ec = exact_pipeline(float(t), variant)
        assert (float(si), float(ci)) == (es, ec), float(t)


# --------------------------------------------------------------------------
# A2 quarter-angle series
# --------------------------------------------------------------------------

def test_series_is_the_printed_polynomial(golden):
    """the oracle's fp32 Horner series equals the printed polynomial
    (exact rational coefficients from the paper's digits) within fp32 Horner rounding."""
    qs = np.linspace(-0.5, 0.5, 2001).astype(np.float32)
    for name, v in (("N", oracle.VARIANT_N), ("A", oracle.VARIANT_A)):
        ss, cc = paper_coeffs(golden, name)
        for q in qs[::7]:
            s, c = oracle.poly_quarter(float(q), v)
            x = Fraction(float(q))
            x2 = x * x
            ps = x * (ss[0] + x2 * (ss[1] + x2 * (ss[2] + x2 * ss[3])))
            pc = 1 + x2 * (cc[0] + x2 * (cc[1] + x2 * cc[2]))
            assert abs(float(Fraction(s) - ps)) < 2.5e-7
            assert abs(float(Fraction(c) - pc)) < 2.5e-7


def test_series_approximates_quarter_angle():
    """method-1 series ~ (sin, cos)(pi x/2); method-2 series
    ratio ~ tan(pi x/2) (fitted to the angle, not a unit pair)."""
    qs = np.linspace(-0.5, 0.5, 4001).astype(np.float32)
    emax_n = emax_a = 0.0
    for q in qs:
        s, c = oracle.poly_quarter(float(q), oracle.VARIANT_N)
        emax_n = max(emax_n, abs(s - math.sin(math.pi * q / 2)), abs(c - math.cos(math.pi * q / 2)))
        s, c = oracle.poly_quarter(float(q), oracle.VARIANT_A)
        emax_a = max(emax_a, abs(math.atan2(s, c) - math.pi * float(q) / 2))
    assert emax_n < 2.5e-7
    assert emax_a < 1.5e-7
    # "do not satisfy sin^2+cos^2=1": raw magnitude at x=1/2 is off by ~6e-4 (SURVEY [X6])
    s, c = oracle.poly_quarter(0.5, oracle.VARIANT_A)
    assert 3e-4 < 1 - math.hypot(s, c) < 1e-3


# --------------------------------------------------------------------------
# A3 doubling (Eq. 1) and its stability analysis
# --------------------------------------------------------------------------

def test_double_angle_closed_forms():
    """CLOSED: (0,1) is fixed; (sin pi/8, cos pi/8) -> (sin pi/4, cos pi/4) within 2 ulp."""
    assert oracle.double_angle(0.0, 1.0) == (0.0, 1.0)
    s, c = oracle.double_angle(float(f32(math.sin(math.pi / 8))), float(f32(math.cos(math.pi / 8))))
    assert abs(s - math.sin(math.pi / 4)) < 2 * 2 ** -24 and abs(c - math.cos(math.pi / 4)) < 2 * 2 ** -24
    s, c = oracle.double_angle(1.0, 0.0)           # quarter turn -> half turn
    assert (s, c) == (0.0, -1.0)


def test_eq1_angle_stable_eq2_mixes_amplitude():
    """with s1 = a sin(t+d), c1 = a cos(t+d), Eq. (1) gives a^2 (sin, cos) 2(t+d)
    (angle stable), Eq. (2) adds (1-a^2) to the cosine (angle and amplitude mixed)."""
    worst1 = worst2 = 0.0
    for a in (0.999, 1.001):
        for t in np.linspace(-1.5, 1.5, 61):
            s0, c0 = float(f32(a * math.sin(t))), float(f32(a * math.cos(t)))
            s1, c1 = oracle.double_angle(s0, c0, oracle.DOUBLING_EQ1)
            s2, c2 = oracle.double_angle(s0, c0, oracle.DOUBLING_EQ2)
            ref = math.atan2(s0, c0) * 2
            d1 = abs(math.remainder(math.atan2(s1, c1) - ref, 2 * math.pi))
            d2 = abs(math.remainder(math.atan2(s2, c2) - ref, 2 * math.pi))
            worst1, worst2 = max(worst1, d1), max(worst2, d2)
            assert abs(math.hypot(s1, c1) - a * a) < 1e-6               # a^2 amplitude
            assert abs(c2 - (a * a * math.cos(2 * math.atan2(s0, c0)) + (1 - a * a))) < 1e-6
    assert worst1 < 1e-6
    assert worst2 > 10 * worst1


def test_eq2_pipeline_is_unstable(golden):
    """PAPER P:94-96, 114 + SURVEY [X14]: the same pipeline with Eq. (2) and an exact final
    renormalisation is far worse with the method-2 coefficients (~2.4e-3) than Eq. (1)."""
    th = np.linspace(-math.pi, math.pi, 20001, dtype=np.float64).astype(np.float32)
    o = oracle.opts(oracle.VARIANT_A)
    o.doubling, o.fix = oracle.DOUBLING_EQ2, oracle.FIX_EXACT_FINAL
    s, c = oracle.sincos(th, o)
    e2 = oracle.error_stats(th, s, c).max_comb
    s, c = oracle.sincos(th, oracle.VARIANT_A)
    e1 = oracle.error_stats(th, s, c).max_comb
    assert e1 < 4.8e-7 * 1.25
    assert 1e-3 < e2 < 5e-3
    assert abs(e2 - golden["survey_crosscheck"]["eq2_instability"]["A_eq2"]) / e2 < 0.05


def test_amplitude_drift_is_2n_times_initial():
    """after n=2 doublings the amplitude error is ~2n = 4 times the
    series' initial amplitude error (a^{2n} ~ 1 + 2n eps)."""
    for q in np.linspace(0.01, 0.5, 50).astype(np.float32):
        s, c = oracle.poly_quarter(float(q), oracle.VARIANT_A)
        eps = math.hypot(s, c) - 1.0                       # large for method 2 (~1e-4)
        sf, cf = oracle.pair_from_q(float(q), oracle.VARIANT_A_NOFIX)
        drift = math.hypot(sf, cf) - 1.0
        assert abs(drift - ((1 + eps) ** 4 - 1)) < 2e-6
        if abs(eps) > 1e-5:
            assert abs(drift / eps - 4) < 0.05


def test_penultimate_fix_identity():
    """PAPER Fig. 1 comment P:320-336: |final| = |penultimate|^2, so 1/|pen|^2 (method 2) or
    2 - |pen|^2 (method 1) corrects the final magnitude to 1 to first order."""
    for q in np.linspace(-0.5, 0.5, 101).astype(np.float32):
        s, c = oracle.pair_from_q(float(q), oracle.VARIANT_A)
        assert abs(math.hypot(s, c) - 1) < 4 * 2 ** -24             # SPEC S:98 "within 4 ULP"
    # the linear fix cannot absorb the method-2 coefficients' large amplitude error (SURVEY [X2])
    th = np.linspace(-math.pi, math.pi, 20001).astype(np.float32)
    s, c = oracle.sincos(th, oracle.VARIANT_A_LINFIX)
    assert oracle.error_stats(th, s, c).max_comb > 1e-6


# --------------------------------------------------------------------------
# end-to-end accuracy vs the paper's figures
# --------------------------------------------------------------------------

@pytest.fixture(scope="module")
def grid_stats():
    return {v: oracle.grid_stats(v, 1 << 24) for v in (oracle.VARIANT_N, oracle.VARIANT_A)}


def test_accuracy_matches_paper(golden, grid_stats):
    """PAPER P:133-139 (N: rms 1.2e-7, max 4.8e-7, amp 1.8e-7) and P:155-157 (A: rms 9.8e-8,
    max 3.8e-7) on [-pi, pi) vs double libm (readings G10, G11: rms within 3%, max within 1.25x)."""
    acc = golden["paper_values"]["accuracy"]
    for name, v in (("N", oracle.VARIANT_N), ("A", oracle.VARIANT_A)):
        st = grid_stats[v]
        assert st.count == 1 << 24 and st.nan_count == 0
        assert abs(st.rms / acc[name]["rms"] - 1) < 0.03, (name, st.rms)
        assert st.max_comb <= 1.25 * acc[name]["max"], (name, st.max_comb)
        assert st.max_amp <= acc["N"]["max_amplitude"], (name, st.max_amp)
    # "a slightly better error budget" for method 2
    assert grid_stats[oracle.VARIANT_A].rms < grid_stats[oracle.VARIANT_N].rms
    assert grid_stats[oracle.VARIANT_A].max_comb < grid_stats[oracle.VARIANT_N].max_comb


def test_grid_matches_independent_transcription(golden, grid_stats):
    """SURVEY [X8]: rms, max, argmax and output sums of the 2^24 grid, bit for bit."""
    x = golden["survey_crosscheck"]["grid_2p24"]
    for name, v in (("N", oracle.VARIANT_N), ("A", oracle.VARIANT_A)):
        st = grid_stats[v]
        assert f"{st.rms:.6e}" == f"{x[name]['rms']:.6e}"
        assert f"{st.max_comb:.6e}" == f"{x[name]['max']:.6e}"
        assert st.worst_bits == int(x[name]["argmax_bits"], 16)
        assert st.sum_s == x[name]["sum_s"]
        assert st.sum_c == x[name]["sum_c"]


def test_fix_variants_and_text_ss2_are_distinguishable(golden, grid_stats):
    """SURVEY [X2]/[X8]: the text final-pair fix, no fix, and the text ss2 each change the
    output bits somewhere -- the grid sums above would catch a swap."""
    th = np.linspace(-math.pi, math.pi, 1 << 16).astype(np.float32)
    base_n = oracle.sincos(th, oracle.VARIANT_N)
    base_a = oracle.sincos(th, oracle.VARIANT_A)
    for v, base in ((oracle.VARIANT_N_TEXTFIX, base_n), (oracle.VARIANT_N_NOFIX, base_n),
                    (oracle.VARIANT_A_TEXT, base_a)):
        s, c = oracle.sincos(th, v)
        assert np.any(s != base[0]) or np.any(c != base[1])
    s, c = oracle.sincos(th, oracle.VARIANT_N_NOFIX)
    st = oracle.error_stats(th, s, c)
    assert st.max_amp > 3e-7            # ~4 LSB-scale drift without the fix


def test_long_double_reference_agrees(golden):
    """LIBM: long-double sinl/cosl and double sin/cos give the same stats to ~7 digits on a
    dense grid, and the oracle stays within the paper-scale bound against both."""
    th = np.linspace(-math.pi, math.pi, 200001).astype(np.float32)
    for v, name in ((oracle.VARIANT_N, "N"), (oracle.VARIANT_A, "A")):
        s, c = oracle.sincos(th, v)
        d = oracle.error_stats(th, s, c, oracle.REF_DOUBLE)
        ld = oracle.error_stats(th, s, c, oracle.REF_LONGDOUBLE)
        assert abs(d.rms - ld.rms) / ld.rms < 1e-6
        assert abs(d.max_comb - ld.max_comb) / ld.max_comb < 1e-6
        assert ld.max_comb <= 1.25 * golden["paper_values"]["accuracy"][name]["max"]


# --------------------------------------------------------------------------
# special values, invariants
# --------------------------------------------------------------------------

def test_special_values(golden):
    """CLOSED + SURVEY [X7]: sin 0 = 0, cos 0 = 1 exactly; NaN/Inf -> NaN pair;
    |x1| >= 2^23 -> (0, 1); subnormals stay gradual (reading G7)."""
    sv = golden["survey_crosscheck"]["special_values"]
    for v in (oracle.VARIANT_N, oracle.VARIANT_A):
        th = np.array([0.0, -0.0, 1e30, -1e30, 3.4e38, 2.0 ** 23 * 2 * math.pi * 1.01, 1.4e-45],
                      dtype=np.float32)
        s, c = oracle.sincos(th, v)
        assert np.all(s == 0) and np.all(c == 1)
        s, c = oracle.sincos(np.array([np.nan, np.inf, -np.inf], dtype=np.float32), v)
        assert np.all(np.isnan(s)) and np.all(np.isnan(c))
    s, c = oracle.sincos(np.array([math.pi / 6], dtype=np.float32), oracle.VARIANT_N)
    assert float(s[0]) == float(f32(sv["pi_over_6_N"]["s"])) and float(c[0]) == float(f32(sv["pi_over_6_N"]["c"]))
    s, _ = oracle.sincos(np.array([fl32_pi()], dtype=np.float32), oracle.VARIANT_N)
    assert float(s[0]) == float(f32(sv["fl32_pi_N_s"]))
    s, _ = oracle.sincos(np.array([fl32_pi()], dtype=np.float32), oracle.VARIANT_A)
    assert abs(float(s[0]) - sv["fl32_pi_A_s"]) < 1e-11
    s, c = oracle.sincos(np.array([1e-40], dtype=np.float32), oracle.VARIANT_N)
    assert float(s[0]) == float(f32(sv["subnormal_1e-40_s"])) and float(c[0]) == 1.0


def test_quadrant_points():
    """CLOSED: [0, pi/2, pi, 3pi/2] -> (0,1), (1,0), (0,-1), (-1,0) within 5e-7."""
    th = np.array([0, math.pi / 2, math.pi, 3 * math.pi / 2], dtype=np.float32)
    for v in (oracle.VARIANT_N, oracle.VARIANT_A):
        s, c = oracle.sincos(th, v)
        np.testing.assert_allclose(s, [0, 1, 0, -1], atol=5e-7)
        np.testing.assert_allclose(c, [1, 0, -1, 0], atol=5e-7)


def test_odd_even_symmetry_by_value():
    """CLOSED: every step is sign-symmetric, so s(-t) = -s(t), c(-t) = c(t) by value
    (signed zero differs: x1 - rint(x1) = +0, reading G6)."""
    rng = np.random.default_rng(3)
    th = np.concatenate([rng.uniform(-1e4, 1e4, 50000), rng.normal(0, 100, 50000),
                         np.float32(10.0) ** rng.uniform(-30, 6, 20000)]).astype(np.float32)
    for v in (oracle.VARIANT_N, oracle.VARIANT_A):
        s, c = oracle.sincos(th, v)
        sn, cn = oracle.sincos(-th, v)
        assert np.array_equal(sn, -s) and np.array_equal(cn, c)


def test_periodicity_exact(golden):
    """CLOSED + SURVEY [X16]: the output depends only on q, so theta' with RN(theta' K) =
    RN(theta K) + k gives bit-identical outputs -- except at x1 = n + 1/2 with odd k, where
    the ties-to-even rule flips q = +-1/2 (the wrap seam)."""
    k32 = np.float32(1 / (2 * math.pi))
    rng = np.random.default_rng(16)
    th = rng.uniform(-100, 100, 3000).astype(np.float32)
    found = 0
    for kk in (1, 3, 17):
        for t in th:
            x1 = np.float32(t * k32)
            target = np.float32(x1 + np.float32(kk))
            if float(target) != float(x1) + kk:
                continue
            u0 = bits(np.float32(float(t) + 2 * math.pi * kk))
            for d in range(-16, 17):
                tp = np.float32(from_bits(u0 + d))
                if np.float32(tp * k32) == target:
                    a = oracle.sincos(np.array([t, tp], dtype=np.float32), oracle.VARIANT_N)
                    assert a[0][0] == a[0][1] and a[1][0] == a[1][1]
                    found += 1
                    break
    assert found > 1000
    # the tie example: x1 = 14.5 -> 15.5 flips q from +1/2 to -1/2
    ex = golden["survey_crosscheck"]["periodicity_tie_example"]
    t = _theta_with_x1(14.5)
    tp = _theta_with_x1(15.5)
    s, _ = oracle.sincos(np.array([t, tp], dtype=np.float32), oracle.VARIANT_N)
    assert s[0] == -s[1] and abs(abs(float(s[0])) - ex["s_abs"]) < 1e-13


def test_smooth_except_at_wrap(golden):
    """no seams except where the reduction wraps at (2n+1) pi.  Mean error over
    4096-float windows in q (SURVEY [X14]): interior jumps tiny, the wrap jump large."""
    # q just inside +1/2 and -1/2 (the wrap) and windows in the interior
    def window_mean(lo_bits, sign):
        q = np.array([sign * from_bits(b) for b in range(lo_bits, lo_bits + 4096)], dtype=np.float32)
        out = []
        for v in (oracle.VARIANT_N,):
            s = np.empty_like(q); c = np.empty_like(q)
            for i, qq in enumerate(q):
                s[i], c[i] = oracle.pair_from_q(float(qq), v)
            ref_s, ref_c = np.sin(2 * np.pi * q.astype(np.float64)), np.cos(2 * np.pi * q.astype(np.float64))
            out.append(np.mean(np.hypot(s - ref_s, c - ref_c)))
        return out[0]
    top = bits(np.float32(0.5)) - 4096
    # the two sides of the wrap: q -> +1/2 and q -> -1/2 land on opposite ends of the seam
    # Signed errors would show the jump; use the sine component directly:
    qs_p = np.array([from_bits(b) for b in range(top, top + 4096)], dtype=np.float32)
    sp = np.array([oracle.pair_from_q(float(x), oracle.VARIANT_N)[0] for x in qs_p[-64:]])
    sm = np.array([oracle.pair_from_q(float(-x), oracle.VARIANT_N)[0] for x in qs_p[-64:]])
    es_p = np.mean(sp - np.sin(2 * np.pi * qs_p[-64:].astype(np.float64)))
    es_m = np.mean(sm - np.sin(-2 * np.pi * qs_p[-64:].astype(np.float64)))
    wrap_jump = abs(es_p - es_m)
    # interior: adjacent windows around q = 0.2
    b0 = bits(np.float32(0.2))
    m1, m2 = window_mean(b0 - 4096, 1.0), window_mean(b0, 1.0)
    interior_jump = abs(m1 - m2)
    sc = golden["survey_crosscheck"]["seams"]
    assert interior_jump < 2 * sc["interior_jump_N"]
    assert wrap_jump > 0.5 * sc["wrap_jump_N"]
    assert wrap_jump > 5 * interior_jump


# --------------------------------------------------------------------------
# exhaustive pins: the argmax chunks (fast) and the committed whole-space run
# --------------------------------------------------------------------------

@pytest.mark.parametrize("name,variant", [("N", oracle.VARIANT_N), ("A", oracle.VARIANT_A),
                                          ("A_text", oracle.VARIANT_A_TEXT)])
def test_exhaustive_maxima_at_their_argmax(golden, name, variant):
    """SURVEY [X5]: the whole-space maxima sit where the independent transcription found them;
    sweep every fp32 pattern within +-2^17 of each argmax (kernel-only q and end-to-end theta)."""
    x = golden["survey_crosscheck"]
    for key, mode in (("exhaustive_q_half", 1), ("exhaustive_theta_0_pi", 0)):
        ref = x[key][name]
        if "argmax" not in ref:
            continue
        b = bits(np.float32(ref["argmax"]))
        top = 0x3F000000 if mode == 1 else 0x40490FDB      # q <= 1/2, theta <= fl32(pi)
        st = oracle.sweep_bits(variant, mode, b - (1 << 17), min(b + (1 << 17), top))
        assert f"{st.max_comb:.4e}" == f"{ref['max']:.4e}", (key, st.max_comb)
        assert st.worst_bits == b, (key, st.worst_x)


def test_committed_exhaustive_run_matches_independent_transcription(golden):
    """SURVEY [X5], [X13] vs tests/golden/oracle_exhaustive.json (written by
    tests/golden/make_oracle_exhaustive.py, oracle only): maxima over all q in [0,1/2] and all
    theta in [0, pi], and the all-2^32 output hash."""
    import json
    import os
    p = os.path.join(os.path.dirname(__file__), "golden", "oracle_exhaustive.json")
    if not os.path.exists(p):
        pytest.skip("run tests/golden/make_oracle_exhaustive.py first")
    run = json.load(open(p))
    x = golden["survey_crosscheck"]
    for name in ("N", "A", "A_text"):
        for key, rk in (("exhaustive_q_half", "q_half"), ("exhaustive_theta_0_pi", "theta_0_pi")):
            ref = x[key][name]
            assert f"{run[name][rk]['max']:.4e}" == f"{ref['max']:.4e}", (name, key)
            if "argmax" in ref:
                assert float(np.float32(run[name][rk]["argmax"])) == float(np.float32(ref["argmax"]))
            if "max_amp" in ref:
                assert f"{run[name][rk]['max_amp']:.4e}" == f"{ref['max_amp']:.4e}", (name, key)
    hb = x["all_bits_hash"]
    for name in ("N", "A"):
        assert run[name]["all_bits"]["hash"] == hb[name]
        assert run[name]["all_bits"]["nan_pairs"] == hb["nan_pairs"]
        assert run[name]["all_bits"]["exact_0_1"] == hb["exact_0_1"]


@pytest.mark.exhaustive
@pytest.mark.parametrize("name,variant", [("N", oracle.VARIANT_N), ("A", oracle.VARIANT_A)])
def test_all_bits_hash_live(golden, name, variant):
    """SURVEY [X13], re-run live (SINCOS_EXHAUSTIVE=1): all 2^32 fp32 inputs."""
    h, nn, ex = oracle.hash_bits(variant, 0, 0xFFFFFFFF)
    hb = golden["survey_crosscheck"]["all_bits_hash"]
    assert "0x%016X" % h == hb[name] and nn == hb["nan_pairs"] and ex == hb["exact_0_1"]


def test_error_stats_interleaved_equals_split_form():
    """oracle.error_stats_interleaved (the {cos, sin} record layout, G13) reports exactly what
    the split form reports on the same pairs -- and that split form is pinned against the
    paper's table above -- including a NaN, an infinity and a wrong pair."""
    rng = np.random.default_rng(5)
    th = np.concatenate([rng.uniform(-1e4, 1e4, 5000), [np.nan, np.inf, 0.0, -0.0]]).astype(np.float32)
    for variant in (oracle.VARIANT_N, oracle.VARIANT_A):
        s, c = oracle.sincos(th, variant)
        s[7] = np.float32(3.0)                       # one wrong pair: it must set max_comb / worst_x
        cs = np.empty(2 * th.size, dtype=np.float32)
        cs[0::2], cs[1::2] = c, s
        for ref in (oracle.REF_DOUBLE, oracle.REF_LONGDOUBLE):
            a = oracle.error_stats(th, s, c, ref).as_dict()
            b = oracle.error_stats_interleaved(th, cs, ref).as_dict()
            assert a == b or all((x == y) or (x != x and y != y) for x, y in zip(a.values(), b.values())), (a, b)
            assert a["worst_x"] == th[7] and a["nan_count"] >= 1
