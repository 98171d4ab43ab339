"""NEXT(3) on the CPU: the oracle's general method (any degrees, doubling count, fix) and the
coefficient regeneration of paper_cs_0406049_b200.coeff_fit, pinned to the paper.

coeff_fit is host-side numpy (double) that produces coefficient tables; the tables are inputs
to both the oracle and the kernel, like the angles."""
import math

import numpy as np
import pytest

import inputs
import oracle
from paper_cs_0406049_b200 import coeff_fit as cf

PAPER_N = (np.array([1.5707963235, -0.645963615, 0.0796819754, -0.0046075748]),
           np.array([-1.2336977925, 0.2536086171, -0.0204391631]))
PAPER_A = (np.array([1.5707963268, -0.6466386396, 0.0679105987, -0.0011573807]),
           np.array([-1.2341299769, 0.2465220241, -0.0123926179]))


@pytest.mark.parametrize("variant", [oracle.VARIANT_N, oracle.VARIANT_A])
def test_general_method_equals_the_paper_pipeline(variant):
    """The general oracle with the paper's tables is the pinned fixed-degree oracle, bit for bit."""
    th = np.concatenate([inputs.generate(2, 0, 200000), inputs.generate(3, 0, 100000)])
    m = oracle.paper_method(variant)
    s1, c1 = oracle.method_sincos(th, m)
    s2, c2 = oracle.sincos(th, variant)
    same = lambda a, b: np.array_equal(a, b) or np.all((a == b) | (np.isnan(a) & np.isnan(b)))  # noqa: E731
    assert same(s1, s2) and same(c1, c2)


def test_general_method_closed_forms():
    """CLOSED: no doublings, s = RN(q*k), c = 1; one doubling of (q*pi, 1 - ...) etc."""
    m = oracle.make_method([2.0], [], doublings=0, fix=oracle.FIX_NONE)
    for q in (0.0, 0.125, -0.25, 0.5):
        assert oracle.method_pair_from_q(q, m) == (2 * q, 1.0)
    # one doubling of the exact pair (0, 1) stays (0, 1); with cc = [-2] and q = 1/2: c1 = 1 - 2/4 = 0.5
    m = oracle.make_method([1.0], [-2.0], doublings=1, fix=oracle.FIX_NONE)
    s, c = oracle.method_pair_from_q(0.5, m)        # s1 = 0.5, c1 = 0.5 -> (2*0.25, 0.25 - 0.25)
    assert (s, c) == (0.5, 0.0)
    with pytest.raises(ValueError):
        oracle.method_pair_from_q(0.1, oracle.make_method([1.0], [], doublings=0, fix=oracle.FIX_RECIPROCAL))


def test_angle_objective_picks_the_fig1_ss2():
    """Reading G1 (SURVEY [X6]): with the other six method-2 coefficients as printed, the
    P:152-154 objective (angle of the raw pair vs the input angle) is minimised at
    ss2 = -0.64663863957..., i.e. Fig. 1's -0.6466386396, not the text's -0.6466386936."""
    start = cf.Fit(PAPER_A[0].copy(), PAPER_A[1].copy(), 2, "angle", 0.0)
    f = cf.fit_angle(free=[("ss", 1)], start=start, points=200001)
    assert abs(f.ss[1] - (-0.6466386396)) < 1e-9
    assert abs(f.ss[1] - (-0.6466386936)) > 5e-8
    x = np.linspace(0, 0.5, 200001)[1:]
    fig1 = np.sqrt(np.mean(cf.angle_residual(PAPER_A[0], PAPER_A[1], 2, x) ** 2))
    text = PAPER_A[0].copy()
    text[1] = -0.6466386936
    assert fig1 < np.sqrt(np.mean(cf.angle_residual(text, PAPER_A[1], 2, x) ** 2)) / 100


def test_paper_method2_is_a_stationary_point_of_its_objective():
    """Gauss-Newton on all seven coefficients, seeded at the printed method-2 table, stays
    close to it (leading terms within 1e-4, the least-determined top terms within 2e-3,
    relative): the table sits at (near) a local optimum of P:153's fit.  Seeded from the
    method-1 fit instead, the same objective lands on a different optimum far away."""
    start = cf.Fit(PAPER_A[0].copy(), PAPER_A[1].copy(), 2, "angle", 0.0)
    f = cf.fit_angle(start=start)
    rel_ss, rel_cc = np.abs(f.ss / PAPER_A[0] - 1), np.abs(f.cc / PAPER_A[1] - 1)
    assert np.all(rel_ss[:3] < 1e-4) and np.all(rel_cc[:2] < 1e-4)
    assert rel_ss[3] < 2e-3 and rel_cc[2] < 2e-3
    assert f.residual_rms < 1e-12
    g = cf.fit_angle()
    assert abs(g.ss[1] / PAPER_A[0][1] - 1) > 0.05 and g.residual_rms < 1e-12


def test_normalized_refit_reproduces_the_paper_table():
    """P:124-126 method 1 (least squares for sine and cosine of theta/4): with relative
    weighting the refit matches the printed table to 2e-10 (ss1) .. 7e-4 (cc3) relative; the
    paper's weighting is unstated (SURVEY [X3]: no weighting reproduces it exactly)."""
    f = cf.fit_normalized(weight="relative")
    tol_ss = [1e-9, 1e-7, 1e-5, 5e-4]
    tol_cc = [2e-6, 1e-4, 2e-3]
    assert np.all(np.abs(f.ss / PAPER_N[0] - 1) < tol_ss)
    assert np.all(np.abs(f.cc / PAPER_N[1] - 1) < tol_cc)
    assert abs(f.ss[0] - math.pi / 2) < 1e-8


@pytest.mark.parametrize("kind", ["normalized", "angle"])
def test_refit_end_to_end_accuracy(kind):
    """SPEC S:211/219 bar: refitted tables (rounded to fp32) keep the kernel-only max error over
    q in [0, 1/2] (every 97th fp32 pattern) within 1.5x the paper's max (4.8e-7)."""
    f = cf.fit_normalized(weight="relative") if kind == "normalized" else cf.fit_angle()
    ss, cc = f.fp32()
    m = oracle.make_method(ss, cc, 2, oracle.FIX_LINEAR_PENULTIMATE if kind == "normalized" else oracle.FIX_RECIPROCAL)
    st = oracle.method_sweep_q(m, stride=97)
    assert st.max_comb <= 1.5 * 4.8e-7 and st.max_amp <= 2.5e-7


def test_more_terms_or_doublings_trade_off():
    """any n works with series refitted for 2 pi x / 2^n.  More series terms lower
    the error; with one doubling fewer the series must cover twice the angle."""
    def err(n, ds, dc, kind):
        f = cf.fit_normalized(n, ds, dc, weight="relative") if kind == "n" else cf.fit_angle(n, ds, dc)
        ss, cc = f.fp32()
        fix = oracle.FIX_LINEAR_PENULTIMATE if kind == "n" else oracle.FIX_RECIPROCAL
        return oracle.method_sweep_q(oracle.make_method(ss, cc, n, fix), stride=211).max_comb
    assert err(2, 5, 4, "n") < err(2, 4, 3, "n")
    assert err(2, 3, 3, "n") > 5 * err(2, 4, 3, "n")          # one term too few for method 1
    assert err(2, 3, 3, "a") < 1.5 * 4.8e-7                   # method 2 tolerates it
    assert err(3, 3, 3, "a") < 1.5 * 4.8e-7                   # a third doubling, lower degree
    assert err(1, 5, 5, "a") < err(2, 4, 3, "a")              # fewer doublings, more terms
