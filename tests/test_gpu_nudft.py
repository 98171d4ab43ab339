"""GPU parity of NEXT(2), sincos_nudft (the fused Huygens / non-uniform Fourier sum), against
the oracle's nudft (same pairs, products and sums in double).  ``pytest -m gpu``.

The pairs are bit-identical to the method; the fused sum rounds differently from the
oracle's double sum, so the bar is the bound the header derives from the arithmetic:
  |out_k - F_k| <= (chunk + 2) 2^-24 sum_j |a_j| + 2^-24 |F_k|."""
import numpy as np
import pytest

import oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_cs_0406049_b200 as sp  # noqa: E402
from paper_cs_0406049_b200 import ab  # noqa: E402  (A/B build)

U = 2.0 ** -24


@pytest.fixture(scope="module", autouse=True)
def cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    yield


def rand_complex(rng, n):
    return (rng.normal(size=n) + 1j * rng.normal(size=n)).astype(np.complex64)


def run(f, t, a, units, variant):
    out = sp.nudft(torch.from_numpy(f).cuda(), torch.from_numpy(t).cuda(), torch.from_numpy(a).cuda(),
                   units=units, variant=variant)
    torch.cuda.synchronize()
    return out.cpu().numpy().astype(np.complex128)


def bound(a, F, nt):
    return (sp.nudft_chunk(nt) + 2) * U * np.abs(a).sum() + U * np.abs(F)


@pytest.mark.parametrize("units", [0, 1])
@pytest.mark.parametrize("variant", [0, 1])
@pytest.mark.parametrize("shape", [(300, 1000), (1, 1), (513, 257), (1024, 5000)])
def test_random_problems_within_bound(units, variant, shape):
    nf, nt = shape
    rng = np.random.default_rng(nf + nt)
    f = rng.uniform(0, 512 if units else 3000, nf).astype(np.float32)
    t = np.sort(rng.uniform(0, 1, nt)).astype(np.float32)
    a = rand_complex(rng, nt)
    got = run(f, t, a, units, variant)
    want = oracle.nudft(f, t, a, units, variant)
    assert np.all(np.abs(got - want) <= bound(a, want, nt))


@pytest.mark.parametrize("units", [0, 1])
@pytest.mark.parametrize("variant", [0, 1])
def test_single_amplitude_is_exactly_the_pair(units, variant):
    """a = e_j0: every product and partial sum is exact, so out_k is the method's pair of
    (f_k, t_j0) bit for bit (the fused path evaluates the same pairs as sincos_phase_grid)."""
    rng = np.random.default_rng(5)
    nf, nt = 700, 3000
    f = rng.uniform(0, 400, nf).astype(np.float32)
    t = rng.uniform(-1, 1, nt).astype(np.float32)
    a = np.zeros(nt, np.complex64)
    a[1234] = 1
    got = run(f, t, a, units, variant)
    s, c = oracle.phase_points(f, np.full(nf, t[1234], np.float32), units, variant)
    assert np.array_equal(got.real, c.astype(np.float64)) and np.array_equal(got.imag, s.astype(np.float64))


def test_uniform_grid_matches_fft():
    """LIBRARY: t_j = j/N in turns, f_k = k -> the DFT; torch.fft on the GPU as the reference,
    within the method's pair error times sum|a| plus the summation bound."""
    N = 4096
    rng = np.random.default_rng(6)
    a = rand_complex(rng, N)
    f = np.arange(N, dtype=np.float32)
    t = (np.arange(N) / N).astype(np.float32)
    got = run(f, t, a, 1, 0)
    want = N * torch.fft.ifft(torch.from_numpy(a.astype(np.complex128)).cuda()).cpu().numpy()
    assert np.all(np.abs(got - want) <= 4.9e-7 * np.abs(a).sum() + bound(a, want, N))


def oracle_nudft_threaded(f, t, a, units, variant, block=256):
    """oracle.nudft over blocks of frequencies on all host threads (per-row numerics unchanged)."""
    import os
    from concurrent.futures import ThreadPoolExecutor
    spans = [(i, min(i + block, f.size)) for i in range(0, f.size, block)]
    with ThreadPoolExecutor(os.cpu_count() or 1) as ex:
        parts = list(ex.map(lambda ab: oracle.nudft(f[ab[0]:ab[1]], t, a, units, variant), spans))
    return np.concatenate(parts)


def run_model_bound(f, t, a, units, variant, chunk):
    """Per-row error bound of the fused sum from its documented arithmetic, evaluated on this
    run's own partial sums (not the worst case): every term enters its fp32 accumulators by
    two single-rounding FMAs in order -- re += ar c; re -= ai s; im += ar s; im += ai c --
    over runs of `chunk` consecutive terms (aligned to multiples of chunk), each run then
    added into fp64, the fp64 total rounded once to fp32.  An FMA's rounding error is at most
    2^-24 of its result, so a run's error is at most 2^-24 times the sum of |partial sum| over
    its steps (to first order; the factor 1.01 covers the second order at <= 2048 steps);
    fp64 adds contribute ~2^-53 of the same sums; the final rounding 2^-24 |F|.  The exact
    partial sums are formed here in fp64 from the oracle's pairs (products of two fp32 values
    are exact in fp64).  Returns (bound per row, F per row from the same fp64 sums)."""
    sp_, cp = oracle.phase_grid(f, t, units, variant)
    s64, c64 = sp_.astype(np.float64), cp.astype(np.float64)
    ar, ai = a.real.astype(np.float64)[None, :], a.imag.astype(np.float64)[None, :]
    m, nt = s64.shape
    nrun = -(-nt // chunk)
    out = []
    for steps in (np.stack([ar * c64, -ai * s64], axis=-1), np.stack([ar * s64, ai * c64], axis=-1)):
        st = np.zeros((m, nrun * chunk, 2))
        st[:, :nt] = steps
        part = np.cumsum(st.reshape(m, nrun, 2 * chunk), axis=-1)      # partials inside each run
        out.append((np.abs(part).sum(axis=(1, 2)), part[:, :, -1].sum(axis=1)))
    (pr, fr), (pi, fi) = out
    F = fr + 1j * fi
    b = 1.01 * U * (pr + pi) + 2.0 ** -50 * (pr + pi)
    return b + U * (np.abs(F) + b), F


@pytest.mark.parametrize("units", [0, 1])
@pytest.mark.parametrize("variant", [0, 1])
def test_c4_scale_per_run_bound(units, variant):
    """The C4 shape (2^15 frequencies x 2^15 jittered times, 2^30 terms, random complex
    amplitudes), 64 sampled k against the oracle within the per-run bound of THIS run's partial
    sums -- ~16x tighter than the worst-case header bound.  Negative control: for every sampled
    k the bound is smaller than the term of median |a_j| would be, so one lost or doubled term
    in any row, tile, chunk or segment fails."""
    nf = nt = 1 << 15
    rng = np.random.default_rng(7)
    f = (512 * rng.random(nf)).astype(np.float32)
    if not units:
        f = (2 * np.pi * f.astype(np.float64)).astype(np.float32)
    t = ((np.arange(nt) + rng.random(nt)) * 2.0 ** -15).astype(np.float32)
    a = rand_complex(rng, nt)
    got = run(f, t, a, units, variant)
    ks = np.unique(np.concatenate([[0, nf - 1], rng.integers(0, nf, 62)]))
    want = oracle.nudft(f[ks], t, a, units, variant)
    b, F = run_model_bound(f[ks], t, a, units, variant, sp.nudft_chunk(nt))
    assert np.allclose(F, want, rtol=0, atol=1e-9 * np.abs(a).sum())     # the model's sums are the oracle's
    err = np.abs(got[ks] - want)
    assert np.all(err <= b), (err / b).max()
    worst = bound(a, want, nt)
    assert np.all(b < worst / 10), (b / worst).max()                       # >= 10x tighter than the header bound
    j_med = int(np.argsort(np.abs(a))[nt // 2])
    assert np.all(np.abs(a[j_med]) > b), (np.abs(a[j_med]), b.max())      # one lost term would fail
    print(f"units {units} variant {variant}: max err/bound {(err / b).max():.3f}, bound {b.max():.3g}, "
          f"median |a_j| {np.abs(a[j_med]):.3f}")


@pytest.mark.parametrize("units,variant", [(0, 0), (0, 1), (1, 0), (1, 1)])
def test_c4_every_row_within_its_per_run_bound(units, variant):
    """All 2^15 outputs at the C4 shape (not a sample): each within the per-run bound of its own
    partial sums, against the oracle's fp64 sum -- rows evaluated in blocks on all host threads
    (~6 s per case on the GPU box's host)."""
    import os
    from concurrent.futures import ThreadPoolExecutor
    nf = nt = 1 << 15
    rng = np.random.default_rng(17 + units)
    f = (512 * rng.random(nf)).astype(np.float32)
    if not units:
        f = (2 * np.pi * f.astype(np.float64)).astype(np.float32)
    t = ((np.arange(nt) + rng.random(nt)) * 2.0 ** -15).astype(np.float32)
    a = rand_complex(rng, nt)
    got = run(f, t, a, units, variant)
    want = oracle_nudft_threaded(f, t, a, units, variant)
    chunk = sp.nudft_chunk(nt)
    blocks = [(r, min(r + 64, nf)) for r in range(0, nf, 64)]
    with ThreadPoolExecutor(os.cpu_count() or 1) as ex:
        bounds = list(ex.map(lambda ab: run_model_bound(f[ab[0]:ab[1]], t, a, units, variant, chunk)[0], blocks))
    b = np.concatenate(bounds)
    err = np.abs(got - want)
    assert np.all(err <= b), (int(np.argmax(err / b)), float((err / b).max()))
    print(f"units {units} variant {variant}: all {nf} rows, max err/bound {(err / b).max():.4f}")


@pytest.mark.parametrize("variant", [0, 1])
@pytest.mark.parametrize("imag", [False, True])
def test_c4_shape_exact_sum(variant, imag):
    """An exact case at the C4 shape (2^15 x 2^15): phases in turns p = RN(f_k m_j / 2) with
    integer f_k in [0, 512) and integer m_j, so q = p - rint(p) is 0 or +-1/2, where the method's
    cosine is exactly +1 or -1 (c = -1 iff f_k and m_j are both odd); small-integer amplitudes,
    all real (or all imaginary).  Then every fp32 partial sum of the real (imaginary) part is a
    small integer -- exact -- and the sum over all 2^15 terms, across every tile, chunk and
    segment boundary, must equal the oracle's (exact, fp64) sum BIT FOR BIT, for every k.  The
    other part (multiples of the tiny sine at q = +-1/2) within the per-run bound."""
    nf = nt = 1 << 15
    rng = np.random.default_rng(11 + variant + 2 * imag)
    f = rng.integers(0, 512, nf).astype(np.float32)
    mj = rng.integers(0, 1 << 15, nt)
    t = (mj / 2.0).astype(np.float32)
    amp = rng.integers(-3, 4, nt).astype(np.float32)
    a = (1j * amp if imag else amp + 0j).astype(np.complex64)
    got = run(f, t, a, 1, variant)
    want = oracle_nudft_threaded(f, t, a, 1, variant)
    ex_got, ex_want = (got.imag, want.imag) if imag else (got.real, want.real)
    assert np.all(ex_want == np.rint(ex_want))                          # the exact part: integers
    assert np.array_equal(ex_got, ex_want.astype(np.float32).astype(np.float64))
    # not degenerate: the parity pattern and the amplitudes make the rows differ
    odd = f.astype(np.int64) % 2 == 1
    assert np.unique(ex_want[odd]).size == 1 and np.unique(ex_want[~odd]).size == 1
    assert ex_want[odd][0] != ex_want[~odd][0]
    ks = np.unique(np.concatenate([[0, nf - 1], rng.integers(0, nf, 30)]))
    b, _ = run_model_bound(f[ks], t, a, 1, variant, sp.nudft_chunk(nt))
    assert np.all(np.abs(got[ks] - want[ks]) <= b)


def test_edges():
    f = torch.rand(10, device="cuda")
    out = torch.full((10,), 7 + 7j, dtype=torch.complex64, device="cuda")
    sp.nudft(f, torch.empty(0, device="cuda"), torch.empty(0, dtype=torch.complex64, device="cuda"), out=out)
    torch.cuda.synchronize()
    assert torch.all(out == 0)
    sp.nudft(torch.empty(0, device="cuda"), torch.rand(5, device="cuda"),
             torch.zeros(5, dtype=torch.complex64, device="cuda"))


@pytest.mark.parametrize("variant", [sp.CMP_LIBM_SINCOSF, sp.CMP_INTRINSIC_SINCOSF])
def test_comparison_variants_run(variant):
    """The bench's comparison kernels (CUDA sincosf / __sincosf in the same fused sum) are sane."""
    rng = np.random.default_rng(8)
    f = rng.uniform(0, 50, 256).astype(np.float32)
    t = rng.uniform(0, 1, 2048).astype(np.float32)
    a = rand_complex(rng, 2048)
    got = run(f, t, a, 1, variant)
    want = oracle.nudft(f, t, a, 1, 0)
    assert np.all(np.abs(got - want) <= 1e-3 * np.abs(a).sum())


# ---- NEXT(3) methods inside the fused sum -------------------------------------------------

@pytest.mark.parametrize("variant", [0, 1])
@pytest.mark.parametrize("units", [0, 1])
def test_nudft_method_with_paper_tables_equals_nudft(variant, units):
    rng = np.random.default_rng(11)
    f = torch.from_numpy(rng.uniform(0, 300, 999).astype(np.float32)).cuda()
    t = torch.from_numpy(rng.uniform(0, 1, 4097).astype(np.float32)).cuda()
    a = torch.from_numpy(rand_complex(rng, 4097)).cuda()
    o1 = sp.nudft(f, t, a, units=units, variant=variant)
    o2 = sp.nudft(f, t, a, units=units, method=sp.make_method(*sp.PAPER_METHODS[variant]))
    torch.cuda.synchronize()
    assert torch.equal(o1, o2)


@pytest.mark.parametrize("units", [0, 1])
@pytest.mark.parametrize("spec", [(1, 3, 2), (2, 3, 3), (3, 3, 3), (1, 6, 5)])
def test_nudft_method_single_amplitude_exact(units, spec):
    """A refitted method (angle fit, reciprocal fix) inside the fused sum: with a = e_j0 the
    outputs are exactly that method's pairs (oracle general method on q = p - rint(p))."""
    from paper_cs_0406049_b200 import coeff_fit as cf
    n, ds, dc = spec
    ss, cc = cf.fit_angle(n, ds, dc).fp32()
    m = sp.make_method(list(ss), list(cc), n, sp.FIX_RECIPROCAL)
    om = oracle.make_method(ss, cc, n, oracle.FIX_RECIPROCAL)
    rng = np.random.default_rng(12)
    f = rng.uniform(0, 300, 700).astype(np.float32)
    t = rng.uniform(-1, 1, 2000).astype(np.float32)
    a = np.zeros(2000, np.complex64)
    a[777] = 1
    got = sp.nudft(torch.from_numpy(f).cuda(), torch.from_numpy(t).cuda(), torch.from_numpy(a).cuda(),
                   units=units, method=m).cpu().numpy()
    p = f * t[777]                                            # fp32 products = RN(f t)
    if units == 0:
        ws, wc = oracle.method_sincos(p, om)
    else:
        q = (p.astype(np.float64) - np.rint(p.astype(np.float64))).astype(np.float32)   # exact
        ws = np.empty_like(q)
        wc = np.empty_like(q)
        for i, qq in enumerate(q):
            ws[i], wc[i] = oracle.method_pair_from_q(float(qq), om)
    assert np.array_equal(got.real, wc) and np.array_equal(got.imag, ws)


# ---- packed fp32 (FFMA2) kernels --------------------------------------------------------

@pytest.mark.parametrize("units", [0, 1])
@pytest.mark.parametrize("kind", ["N", "A", "m1_3_2", "m2_4_3", "g3_3_2", "g2_5_4", "g1_4_4"])
@pytest.mark.parametrize("shape", [(1, 1), (3, 7), (513, 1031), (1500, 4100)])
def test_packed_kernel_bit_identical_to_scalar(units, kind, shape):
    """The packed kernels of the product (two frequencies per FFMA2/FMUL2/FADD2 lane pair) round
    every lane exactly as their scalar twins (the A/B build's nudft_packed = 0) do
    -- the sums are bit-identical, for the paper's tables, the
    specialised method shapes and general shapes, ragged nf (odd lane pairs past nf) and nt
    (tail tiles).
    Phases include exact zeros, half-turn ties and huge / subnormal / non-finite values."""
    nf, nt = shape
    rng = np.random.default_rng(nf * 7 + nt)
    f = rng.uniform(0, 512 if units else 3000, nf).astype(np.float32)
    t = rng.uniform(-1, 1, nt).astype(np.float32)
    special = np.array([0.0, -0.0, 0.5, 1.5, 2.5, -0.5, 1e-40, -1e-45, 3e30, np.inf, -np.inf, np.nan],
                       np.float32)
    f[: min(nf, special.size)] = special[: min(nf, special.size)]
    t[: min(nt, 3)] = np.array([1.0, 0.25, 0.5], np.float32)[: min(nt, 3)]
    a = rand_complex(rng, nt)
    if kind in ("N", "A"):
        kw = {"variant": 0 if kind == "N" else 1}
    else:
        from paper_cs_0406049_b200 import coeff_fit as cf
        n, ds, dc = (int(x) for x in kind[1:].split("_"))
        ss, cc = cf.fit_angle(n, ds, dc).fp32()
        # m*: the compile-time shapes; g*: general shapes (run-time doubling loop, zero-padded
        # Horner of 4 or 8 terms), fix reciprocal / linear / none
        fix = {"m1_3_2": sp.FIX_RECIPROCAL, "m2_4_3": sp.FIX_LINEAR, "g3_3_2": sp.FIX_RECIPROCAL,
               "g2_5_4": sp.FIX_LINEAR, "g1_4_4": sp.FIX_NONE}[kind]
        kw = {"method": sp.make_method(list(ss), list(cc), n, fix)}
    fd, td, ad = (torch.from_numpy(x).cuda() for x in (f, t, a))
    with ab.knobs(nudft_packed=0):
        o_scalar = sp.nudft(fd, td, ad, units=units, **kw)
    o_packed = sp.nudft(fd, td, ad, units=units, **kw)
    torch.cuda.synchronize()
    x, y = o_scalar.cpu().numpy(), o_packed.cpu().numpy()
    xb = x.view(np.uint32).reshape(-1, 2)
    yb = y.view(np.uint32).reshape(-1, 2)
    fin = np.isfinite(x.real) & np.isfinite(x.imag)
    assert np.array_equal(fin, np.isfinite(y.real) & np.isfinite(y.imag))
    assert np.array_equal(xb[fin], yb[fin])


def test_ab_knobs_reject_bad_values():
    assert ab.lib().sincos_ab_set(7, 2) == -1 and ab.lib().sincos_ab_set(99, 0) == -1
    assert ab.lib().sincos_ab_get(7) == 1


@pytest.mark.parametrize("variant", [0, 1])
def test_packed_method_equals_scalar_on_all_fp32_inputs(variant):
    """Exhaustive form of the packed/scalar identity: the two-lane method (FFMA2/FMUL2/FADD2)
    equals the scalar method bit for bit on every one of the 2^32 fp32 inputs, in radians
    (scale by 1/2pi first) and in turns -- the phases the fused sum feeds it are a subset."""
    assert sp.debug_packed_check(variant) == 0


@pytest.mark.parametrize("spec", [(2, 4, 3, 0), (2, 4, 3, 1), (1, 3, 2, 0), (1, 3, 2, 1)])
def test_packed_method_shapes_equal_scalar_on_all_fp32_inputs(spec):
    from paper_cs_0406049_b200 import coeff_fit as cf
    n, ds, dc, fix = spec
    ss, cc = cf.fit_angle(n, ds, dc).fp32()
    assert sp.debug_packed_check(method=sp.make_method(list(ss), list(cc), n, fix)) == 0


def test_packed_check_negative_control_fails():
    """The exhaustive check can fail: packed method 1 against scalar method 2 differs wherever
    the two tables give different pairs (every q not tiny and not 0: roughly the patterns with
    1e-4 < |x| < 2^23 turns, ~15% of all 2^32, x 2 units x 2 components)."""
    assert sp.debug_packed_check(-1) > 2 ** 30


def test_very_long_sum_chunking():
    """nt beyond 65535 x 1024 terms (the grid's y extent at one fp32 run per segment): segments
    hold several runs; a single unit amplitude far down the sum still returns exactly that
    term's pair (every partial sum is exact)."""
    nt = (1 << 26) + (1 << 25) + 77            # 100.7 M terms
    assert sp.nudft_chunk(nt) == 1024
    f = torch.tensor([0.0, 1.0, 3.25, 77.5], device="cuda")
    t = torch.rand(nt, device="cuda")
    a = torch.zeros(nt, dtype=torch.complex64, device="cuda")
    j0 = nt - 5
    a[j0] = 1
    out = sp.nudft(f, t, a, units=sp.TURNS).cpu().numpy()
    p = (f.cpu().numpy() * t[j0].cpu().numpy()).astype(np.float32)        # RN(f t0)
    q = (p.astype(np.float64) - np.rint(p.astype(np.float64))).astype(np.float32)
    want = np.array([oracle.pair_from_q(float(x), 0) for x in q])
    assert np.array_equal(out.real.astype(np.float32), want[:, 1].astype(np.float32))
    assert np.array_equal(out.imag.astype(np.float32), want[:, 0].astype(np.float32))


def test_workspace_alignment_and_size_checked():
    """The fp64 partials need a 16-B aligned workspace of sincos_nudft_workspace_bytes(nf, nt):
    an 8-B offset or one byte short is INVALID_ARGUMENT, not a fault."""
    f = torch.rand(100, device="cuda")
    t = torch.rand(5000, device="cuda")
    a = torch.randn(5000, dtype=torch.complex64, device="cuda")
    need = sp.lib().sincos_nudft_workspace_bytes(100, 5000)
    ws = torch.empty(need + 64, dtype=torch.uint8, device="cuda")
    sp.nudft(f, t, a, workspace=ws[16:16 + need])                 # 16-B aligned: fine
    for bad in (ws[8:8 + need], ws[:need - 1]):
        with pytest.raises(sp.SincosError):
            sp.nudft(f, t, a, workspace=bad)
