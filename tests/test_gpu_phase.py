"""GPU parity of NEXT(1), sincos_phase_grid (pairs of phases f_i * t_j formed in the kernel),
against the oracle's phase functions: bit-exact by value.  ``pytest -m gpu``."""
import contextlib
import numpy as np
import pytest

import inputs
import oracle
from helpers import assert_parity

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_cs_0406049_b200 as sp  # noqa: E402
from paper_cs_0406049_b200 import ab  # noqa: E402  (A/B build)

R, T = 0, 1
COMBOS = [(u, v) for u in (R, T) for v in (0, 1)]


@pytest.fixture(scope="module", autouse=True)
def cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    yield


def c4_axes(nf=1 << 15, nt=1 << 15, turns=False):
    """BASELINE configs[3] axes: f_i = 512 u(3,0,i), t_j = (j + u(3,1,j)) 2^-15 (jittered,
    sorted); in radians the row factor is fl32(2 pi f_i)."""
    f = np.array([512.0 * inputs.urand(3, 0, i) for i in range(nf)])
    t = np.array([(j + inputs.urand(3, 1, j)) * 2.0 ** -15 for j in range(nt)])
    if not turns:
        f = 2 * np.pi * f
    return f.astype(np.float32), t.astype(np.float32)


@pytest.mark.parametrize("units,variant", COMBOS)
@pytest.mark.parametrize("shape", [(37, 53), (100, 1024), (3, 8), (1, 1), (5, 7)])
@pytest.mark.parametrize("inter", [False, True])
def test_small_grids_full(units, variant, shape, inter):
    nf, nt = shape
    rng = np.random.default_rng(nf * 1000 + nt)
    f = rng.uniform(0, 400, nf).astype(np.float32)
    t = rng.uniform(-1, 1, nt).astype(np.float32)
    ws, wc = oracle.phase_grid(f, t, units, variant)
    fd, td = torch.from_numpy(f).cuda(), torch.from_numpy(t).cuda()
    if inter:
        o = torch.empty(2 * nf * nt, device="cuda")
        sp.phase_grid(fd, td, interleaved_out=o, units=units, variant=variant)
        o = o.cpu().numpy()
        gs, gc = o[1::2], o[0::2]
    else:
        s = torch.empty(nf * nt, device="cuda")
        c = torch.empty(nf * nt, device="cuda")
        sp.phase_grid(fd, td, s, c, units=units, variant=variant)
        gs, gc = s.cpu().numpy(), c.cpu().numpy()
    assert_parity(gs, gc, ws.ravel(), wc.ravel(), f"phase {shape} units={units} v={variant}")


@pytest.mark.parametrize("units,variant", COMBOS)
def test_misaligned_outputs_use_the_scalar_path(units, variant):
    nf, nt = 64, 256
    rng = np.random.default_rng(9)
    f = rng.uniform(0, 400, nf).astype(np.float32)
    t = rng.uniform(0, 1, nt).astype(np.float32)
    ws, wc = oracle.phase_grid(f, t, units, variant)
    fd, td = torch.from_numpy(f).cuda(), torch.from_numpy(t).cuda()
    big = torch.empty(2 * nf * nt + 8, device="cuda")
    s, c = big[1:1 + nf * nt], big[nf * nt + 3:2 * nf * nt + 3]
    sp.phase_grid(fd, td, s, c, units=units, variant=variant)
    assert_parity(s.cpu().numpy(), c.cpu().numpy(), ws.ravel(), wc.ravel(), "misaligned")
    tbig = torch.empty(nt + 1, device="cuda")
    tbig[1:] = td
    s2, c2 = torch.empty(nf * nt, device="cuda"), torch.empty(nf * nt, device="cuda")
    sp.phase_grid(fd, tbig[1:], s2, c2, units=units, variant=variant)       # t not 32-B aligned
    assert_parity(s2.cpu().numpy(), c2.cpu().numpy(), ws.ravel(), wc.ravel(), "misaligned t")


@pytest.mark.parametrize("units,variant", COMBOS)
def test_c4_full_size_sampled(units, variant):
    """The C4 shape (2^15 x 2^15 = 2^30 pairs, interleaved, 8 GiB) at full size; ~1M sampled
    elements and whole first/last rows against the oracle's pointwise phase pairs."""
    nf = nt = 1 << 15
    f, t = c4_axes(nf, nt, turns=units == T)
    fd, td = torch.from_numpy(f).cuda(), torch.from_numpy(t).cuda()
    o = torch.empty(2 * nf * nt, device="cuda")
    sp.phase_grid(fd, td, interleaved_out=o, units=units, variant=variant)
    torch.cuda.synchronize()
    rng = np.random.default_rng(units * 2 + variant)
    idx = np.unique(np.concatenate([np.arange(nt), np.arange(nf * nt - nt, nf * nt),
                                    rng.integers(0, nf * nt, 1 << 20)])).astype(np.int64)
    ov = o.view(-1, 2)[torch.from_numpy(idx).cuda()].cpu().numpy()
    ws, wc = oracle.phase_points(f[idx // nt], t[idx % nt], units, variant)
    assert_parity(ov[:, 1].copy(), ov[:, 0].copy(), ws, wc, "C4 phase grid")
    del o
    torch.cuda.empty_cache()


@pytest.mark.parametrize("variant", [0, 1])
def test_radians_equals_the_materialised_path(variant):
    """Product-level consistency: the fused grid in radians equals sincos_pairs on the
    materialised fp32 outer product (torch fp32 multiply = RN(f t)), bit for bit."""
    f, t = c4_axes(1 << 10, 1 << 12)
    fd, td = torch.from_numpy(f).cuda(), torch.from_numpy(t).cuda()
    th = torch.outer(fd, td).reshape(-1).contiguous()
    s1, c1 = sp.sincos(th, variant=variant)
    s2, c2 = torch.empty_like(th), torch.empty_like(th)
    sp.phase_grid(fd, td, s2, c2, units=R, variant=variant)
    torch.cuda.synchronize()
    assert torch.equal(s1, s2) and torch.equal(c1, c2)


@pytest.mark.parametrize("units,variant", COMBOS)
@pytest.mark.parametrize("mode", [1, 3, 0])
def test_ragged_rows_flat_path(units, variant, mode):
    """Rows that are not whole 256-bit vectors (nt % 8 != 0, t or outputs off 32 B) go through
    the row kernel (nt >= 1024: t windows re-aligned per row class) or the short-row kernel
    (8 <= nt < 1024: t from shared memory), the flat kernel (8
    consecutive pairs of the row-major grid per thread, rows wrapping inside a vector, nt = 1..9
    included; for every nt in the A/B build's realign = 3) or, with both disabled / for outputs they
    cannot serve, one pair per thread; bit-exact either way, at several output offsets, split
    and interleaved."""
    rng = np.random.default_rng(31 + units + 2 * variant)
    # mode 1: the product; 3 (flat kernel) and 0 (one pair per thread): the A/B build
    with (contextlib.nullcontext() if mode == 1 else ab.knobs(realign=mode)):
        for nf, nt in ((1, 1), (3, 1), (7, 2), (5, 3), (9, 7), (4, 9), (33, 1001), (257, 255), (64, 256), (5, 127),
                       (6, 129), (2, 5000)):
            f = rng.uniform(0, 400, nf).astype(np.float32)
            t = rng.uniform(-1, 1, nt + 1).astype(np.float32)
            n = nf * nt
            for toff in (0, 1):
                tt = t[toff:toff + nt]
                ws, wc = oracle.phase_grid(f, tt, units, variant)
                ws, wc = ws.ravel(), wc.ravel()
                fd = torch.from_numpy(f).cuda()
                tbig = torch.from_numpy(t).cuda()
                td = tbig[toff:toff + nt]
                for oo, oc in ((0, 0), (3, 3), (5, 5), (1, 2)):
                    big_s = torch.empty(n + 16, device="cuda")
                    big_c = torch.empty(n + 16, device="cuda")
                    s, c = big_s[oo:oo + n], big_c[oc:oc + n]
                    sp.phase_grid(fd, td, s, c, units=units, variant=variant)
                    big_i = torch.empty(2 * n + 16, device="cuda")
                    io = big_i[oo:oo + 2 * n]
                    sp.phase_grid(fd, td, interleaved_out=io, units=units, variant=variant)
                    torch.cuda.synchronize()
                    tag = f"({nf},{nt}) toff={toff} out={oo},{oc} mode={mode}"
                    assert_parity(s.cpu().numpy(), c.cpu().numpy(), ws, wc, "split " + tag)
                    iv = io.cpu().numpy()
                    assert_parity(iv[1::2], iv[0::2], ws, wc, "inter " + tag)


@pytest.mark.parametrize("units,variant", COMBOS)
@pytest.mark.parametrize("nt", [9, 17, 131, 1001, 1024, 1025, 1026, 1027, 1028, 1029, 1030, 1031])
def test_row_path_every_alignment(units, variant, nt):
    """The ragged-row kernels at every t offset x every output offset x nt mod 8, with nf = 19
    rows, split and interleaved: bit-exact vs the oracle.  nt >= 1024: the row kernel (its
    re-alignment K = 0..7, every row class, more rows than classes); 8 <= nt < 1024: the
    short-row kernel (t windows from shared memory, rows wrapping inside a vector)."""
    rng = np.random.default_rng(nt * 7 + units + 2 * variant)
    nf = 19
    n = nf * nt
    f = rng.uniform(0, 400, nf).astype(np.float32)
    t = rng.uniform(-1, 1, nt + 8).astype(np.float32)
    fd, tbig = torch.from_numpy(f).cuda(), torch.from_numpy(t).cuda()
    big_s = torch.empty(n + 16, device="cuda")
    big_c = torch.empty(n + 16, device="cuda")
    big_i = torch.empty(2 * n + 16, device="cuda")
    for toff in range(8):
        ws, wc = oracle.phase_grid(f, t[toff:toff + nt], units, variant)
        ws, wc = ws.ravel(), wc.ravel()
        td = tbig[toff:toff + nt]
        for oo in range(8):
            s, c = big_s[oo:oo + n], big_c[oo:oo + n]
            sp.phase_grid(fd, td, s, c, units=units, variant=variant)
            io = big_i[2 * (oo % 4):2 * (oo % 4) + 2 * n]
            sp.phase_grid(fd, td, interleaved_out=io, units=units, variant=variant)
            tag = f"({nf},{nt}) toff={toff} out={oo}"
            assert_parity(s.cpu().numpy(), c.cpu().numpy(), ws, wc, "split " + tag)
            iv = io.cpu().numpy()
            assert_parity(iv[1::2], iv[0::2], ws, wc, "inter " + tag)


@pytest.mark.parametrize("inter", [False, True])
@pytest.mark.parametrize("shape", [(70001, 131), (2_240_032, 521), (70001, 1029), (2_150_000, 1031)])
def test_row_path_many_rows(inter, shape):
    """Many rows: (70001, 131), (2 240 032, 521) -- the short-row kernel's grid-stride loop;
    (70001, 1029) -- the row kernel past the 65528-block grid height's rows; (2 150 000, 1031)
    -- slot count capped, > 32 rows per slot (f re-loaded per 32-row chunk), 2.2e9 pairs.
    Row i depends on f_i and t only, so sampled rows (the first and
    last, rows around the slot-count multiples, random rows) are compared with the oracle's
    grid of those f values: bit-exact."""
    nf, nt = shape
    rng = np.random.default_rng(77 + nt)
    f = rng.uniform(0, 400, nf).astype(np.float32)
    tb = rng.uniform(-1, 1, nt + 1).astype(np.float32)
    t = tb[1:]                                            # t off 32 B: re-aligned windows
    fd = torch.from_numpy(f).cuda()
    td = torch.from_numpy(tb).cuda()[1:]
    n = nf * nt
    rows = np.unique(np.concatenate([[0, 1, 2, nf - 2, nf - 1], rng.integers(0, nf, 3000),
                                     *[np.arange(k - 9, k + 9) for k in (65528, 262112, 524224, 2 * 262112, 32 * 65528)
                                       if k + 9 < nf]]))
    ws, wc = oracle.phase_grid(f[rows], t, R, 1)
    ri = torch.from_numpy(rows).cuda()
    if inter:
        o = torch.empty(2 * n, device="cuda")
        sp.phase_grid(fd, td, interleaved_out=o, units=R, variant=1)
        o = o.view(nf, nt, 2)[ri].cpu().numpy()
        gs, gc = o[..., 1], o[..., 0]
        del o
    else:
        s, c = torch.empty(n, device="cuda"), torch.empty(n, device="cuda")
        sp.phase_grid(fd, td, s, c, units=R, variant=1)
        gs, gc = s.view(nf, nt)[ri].cpu().numpy(), c.view(nf, nt)[ri].cpu().numpy()
        del s, c
    assert_parity(gs.ravel(), gc.ravel(), ws.ravel(), wc.ravel(), f"({nf},{nt}) inter={inter}")


@pytest.mark.parametrize("variant", [0, 1])
@pytest.mark.parametrize("inter", [False, True])
@pytest.mark.parametrize("config", [1, 3, 5])
def test_sincos_turns(variant, inter, config):
    """sincos_turns(x): the method on angles given in turns, from the reduction on -- the
    oracle's phase pairs with f = 1 in turns; BASELINE generators (read as turns), the C3 edge
    set included, a ragged length (flat kernel) and a multiple of 8 (row kernel)."""
    for n in ((1 << 18) + 3, 1 << 18):
        x = inputs.generate(config, 7, n)
        xd = torch.from_numpy(x).cuda()
        ws, wc = oracle.phase_points(np.ones_like(x), x, T, variant)
        if inter:
            o = sp.sincos_turns(xd, variant=variant, interleaved=True).cpu().numpy()
            gs, gc = o[:, 1], o[:, 0]
        else:
            s, c = sp.sincos_turns(xd, variant=variant)
            gs, gc = s.cpu().numpy(), c.cpu().numpy()
        assert_parity(gs, gc, ws, wc, f"turns config={config} n={n}")


@pytest.mark.parametrize("units,variant", COMBOS)
@pytest.mark.parametrize("nt", [1, 2, 3, 4, 7])
def test_tiny_rows(units, variant, nt):
    """Rows of 1..7 pairs with 32-B aligned outputs: the tiny-row kernel (nt = 1; nt = 2, 3 split:
    groups of 8 rows per thread, static (row, column) per pair, f as one 256-bit load when
    32-B aligned, else scalar) and the short-row kernel for the rest -- whole groups, a ragged
    remainder of < 8 rows, f at an aligned and an unaligned offset."""
    rng = np.random.default_rng(nt * 10 + units + 2 * variant)
    for nf in (8, 13, 1001, 8 * 40_000 + 5):
        fb = rng.uniform(-400, 400, nf + 8).astype(np.float32)
        t = rng.uniform(-1, 1, nt).astype(np.float32)
        n = nf * nt
        for foff in (0, 1):
            f = fb[foff:foff + nf]
            ws, wc = oracle.phase_grid(f, t, units, variant)
            ws, wc = ws.ravel(), wc.ravel()
            fbig = torch.from_numpy(fb).cuda()
            fd, td = fbig[foff:foff + nf], torch.from_numpy(t).cuda()
            s, c = torch.empty(n, device="cuda"), torch.empty(n, device="cuda")
            io = torch.empty(2 * n, device="cuda")
            sp.phase_grid(fd, td, s, c, units=units, variant=variant)
            sp.phase_grid(fd, td, interleaved_out=io, units=units, variant=variant)
            torch.cuda.synchronize()
            tag = f"nt={nt} nf={nf} foff={foff}"
            assert_parity(s.cpu().numpy(), c.cpu().numpy(), ws, wc, "split " + tag)
            iv = io.cpu().numpy()
            assert_parity(iv[1::2], iv[0::2], ws, wc, "inter " + tag)


@pytest.mark.parametrize("nt", [2, 3, 4, 5, 6, 7, 8, 9, 11, 12, 13, 14, 15, 16])
@pytest.mark.parametrize("variant", [0, 1])
@pytest.mark.parametrize("units", [0, 1])
def test_staged_rows(units, variant, nt):
    """Rows of 2..15 pairs through the staged short-row kernel (split nt = 4..14: 4 rows per lane,
    64-thread blocks for 12-13, 2 rows per lane for 14; interleaved nt = 2..15: 4 rows per lane
    up to 7, 2 above; nt = 16 and split 15 on the short-row kernel);
    outputs 16-B aligned at pair 0: a warp's 128 rows staged in shared memory, written back as
    contiguous 128-bit stores): whole 128-row regions and a ragged tail, f 16-B aligned or not,
    outputs 32-B and only 16-B aligned, and on the A/B build's grid-stride grids (many regions
    per warp).  Also the layouts that must not take it (interleaved pairs only 8-B aligned)."""
    rng = np.random.default_rng(1000 + nt * 10 + units + 2 * variant)
    sizes = (127, 128, 129, 128 * 37 + 77, 128 * 2500)
    NF = max(sizes)
    fb = rng.uniform(-400, 400, NF + 8).astype(np.float32)
    t = rng.uniform(-1, 1, nt).astype(np.float32)
    fbig, td = torch.from_numpy(fb).cuda(), torch.from_numpy(t).cuda()
    sb = torch.empty(NF * nt + 16, device="cuda")
    cb = torch.empty(NF * nt + 16, device="cuda")
    ib = torch.empty(2 * NF * nt + 16, device="cuda")
    for ctx in (contextlib.nullcontext(), ab.knobs(blocks_per_sm=1)):
        with ctx:
            for nf in sizes:
                for foff in (0, 1, 4):
                    f = fb[foff:foff + nf]
                    ws, wc = oracle.phase_grid(f, t, units, variant)
                    ws, wc = ws.ravel(), wc.ravel()
                    fd = fbig[foff:foff + nf]
                    n = nf * nt
                    for ooff in (0, 4, 2):          # 32-B / 16-B aligned (staged) / 8-B (short-row kernel)
                        s, c = sb[ooff:ooff + n], cb[ooff:ooff + n]
                        io = ib[ooff:ooff + 2 * n]
                        s.fill_(float("nan")); c.fill_(float("nan")); io.fill_(float("nan"))
                        sp.phase_grid(fd, td, s, c, units=units, variant=variant)
                        sp.phase_grid(fd, td, interleaved_out=io, units=units, variant=variant)
                        torch.cuda.synchronize()
                        tag = f"nt={nt} nf={nf} foff={foff} ooff={ooff}"
                        assert_parity(s.cpu().numpy(), c.cpu().numpy(), ws, wc, "split " + tag)
                        iv = io.cpu().numpy()
                        assert_parity(iv[1::2], iv[0::2], ws, wc, "inter " + tag)


@pytest.mark.parametrize("variant", [0, 1])
@pytest.mark.parametrize("units", [0, 1])
def test_every_row_kernel_on_special_values(units, variant):
    """Every phase-grid kernel (tiny, staged with 4 and 2 rows per lane, short-row, row, vector,
    one pair per thread) on f and t holding the special values -- +-0, subnormals, +-inf, NaN,
    huge, ties of the turn reduction -- so the products RN(f t) are zeros, subnormals, infinities,
    NaN (0 x inf) and exact halves: the outputs equal the oracle's pairs by value (NaN == NaN)."""
    rng = np.random.default_rng(7 + units + 2 * variant)
    specials = np.array([0.0, -0.0, 1e-40, -1e-40, np.inf, -np.inf, np.nan, 3e38, -3e38, 0.5, -0.5, 2.5,
                         1.0, 0.25, 1e30, 7.0], dtype=np.float32)
    for nt, toff, ooff in ((1, 0, 0), (3, 0, 0), (5, 0, 4), (12, 0, 0), (14, 0, 4), (33, 1, 0), (1003, 0, 0),
                           (256, 0, 0), (9, 0, 1)):
        nf = 700
        f = rng.uniform(-50, 50, nf).astype(np.float32)
        f[rng.integers(0, nf, 60)] = rng.choice(specials, 60)
        t = rng.uniform(-2, 2, nt).astype(np.float32)
        t[rng.integers(0, nt, max(1, nt // 4))] = rng.choice(specials, max(1, nt // 4))
        ws, wc = oracle.phase_grid(f, t, units, variant)
        ws, wc = ws.ravel(), wc.ravel()
        fd = torch.from_numpy(f).cuda()
        tb = torch.empty(nt + 8, device="cuda")
        tb[toff:toff + nt].copy_(torch.from_numpy(t))
        td = tb[toff:toff + nt]
        n = nf * nt
        sb, cb, ib = (torch.empty(n + 8, device="cuda"), torch.empty(n + 8, device="cuda"),
                      torch.empty(2 * n + 8, device="cuda"))
        s, c, io = sb[ooff:ooff + n], cb[ooff:ooff + n], ib[ooff:ooff + 2 * n]
        sp.phase_grid(fd, td, s, c, units=units, variant=variant)
        sp.phase_grid(fd, td, interleaved_out=io, units=units, variant=variant)
        torch.cuda.synchronize()
        tag = f"nt={nt} toff={toff} ooff={ooff}"
        assert_parity(s.cpu().numpy(), c.cpu().numpy(), ws, wc, "split " + tag)
        iv = io.cpu().numpy()
        assert_parity(iv[1::2], iv[0::2], ws, wc, "inter " + tag)


@pytest.mark.parametrize("units", [0, 1])
def test_phase_grid_unshared_output_alignment(units):
    """Split outputs with cos[] at every float offset from sin[]'s 32-B frame, and interleaved
    pairs only 4-B aligned (odd float offsets), for short, ragged and long rows: the flat kernel
    with the re-aligned stream written by warp shuffles; raw bits equal the oracle's grid,
    sentinel guard zones around every output."""
    SENT = 0x7F8ABCDE
    G = 64
    bad = []
    for nt, nf in ((1, 3001), (2, 1503), (5, 701), (8, 389), (13, 257), (300, 11), (1001, 4)):
        f = (inputs.generate(1, 0, nf) * np.float32(3.0)).astype(np.float32)
        t = (inputs.generate(2, 7, nt) * np.float32(1e-3)).astype(np.float32)
        fd, td = torch.from_numpy(f).cuda(), torch.from_numpy(t).cuda()
        n = nf * nt
        for variant in (0, 1):
            ws, wc = oracle.phase_grid(f, t, units, variant)
            ws_i = torch.from_numpy(ws.reshape(-1).view(np.int32)).cuda()
            wc_i = torch.from_numpy(wc.reshape(-1).view(np.int32)).cuda()
            bs = torch.empty(2 * G + n + 8, dtype=torch.int32, device="cuda")
            bc = torch.empty_like(bs)
            for os_ in (0, 3):
                for oc in range(8):
                    if (oc - os_) % 8 == 0:
                        continue                    # shared alignment: the other kernels
                    bs.fill_(SENT)
                    bc.fill_(SENT)
                    sp.phase_grid(fd, td, sin_out=bs[G + os_:G + os_ + n].view(torch.float32),
                                  cos_out=bc[G + oc:G + oc + n].view(torch.float32), units=units, variant=variant)
                    ok = (torch.equal(bs[G + os_:G + os_ + n], ws_i) and torch.equal(bc[G + oc:G + oc + n], wc_i) and
                          bool((bs[:G + os_] == SENT).all()) and bool((bs[G + os_ + n:] == SENT).all()) and
                          bool((bc[:G + oc] == SENT).all()) and bool((bc[G + oc + n:] == SENT).all()))
                    if not ok:
                        bad.append(("split", nt, variant, os_, oc))
            bi = torch.empty(2 * G + 2 * n + 8, dtype=torch.int32, device="cuda")
            for oi in (1, 3, 5, 7):
                bi.fill_(SENT)
                sp.phase_grid(fd, td, interleaved_out=bi[G + oi:G + oi + 2 * n].view(torch.float32), units=units,
                              variant=variant)
                got = bi[G + oi:G + oi + 2 * n]
                ok = (torch.equal(got[1::2], ws_i) and torch.equal(got[0::2], wc_i) and
                      bool((bi[:G + oi] == SENT).all()) and bool((bi[G + oi + 2 * n:] == SENT).all()))
                if not ok:
                    bad.append(("inter", nt, variant, oi))
    assert not bad, f"{len(bad)} failing, first {bad[:8]}"
