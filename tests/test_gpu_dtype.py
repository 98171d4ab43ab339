"""GPU parity of NEXT(4): 16-bit outputs (IEEE binary16, bfloat16) and the split <-> interleaved
adapters.  The 16-bit values must equal the oracle's fp32 pair rounded to nearest even by a
library conversion (numpy float16, torch bfloat16 on the CPU).  ``pytest -m gpu``."""
import contextlib
import numpy as np
import pytest

import inputs
import oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_cs_0406049_b200 as sp  # noqa: E402
from paper_cs_0406049_b200 import ab  # noqa: E402  (A/B build)


@pytest.fixture(scope="module", autouse=True)
def cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    yield


def rn16(x: np.ndarray, dtype) -> np.ndarray:
    """The oracle's fp32 values rounded to 16 bits (RN-even) by a library, as uint16 bits."""
    if dtype == torch.float16:
        return x.astype(np.float16).view(np.uint16)
    return torch.from_numpy(x).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)


def same16(got: np.ndarray, want: np.ndarray, dtype) -> np.ndarray:
    g = torch.from_numpy(got.view(np.int16)).view(dtype).float().numpy()
    w = torch.from_numpy(want.view(np.int16)).view(dtype).float().numpy()
    return (got == want) | (np.isnan(g) & np.isnan(w)) | ((g == 0) & (w == 0))


@pytest.mark.parametrize("dtype", [torch.float16, torch.bfloat16])
@pytest.mark.parametrize("variant", [0, 1])
@pytest.mark.parametrize("inter", [False, True])
@pytest.mark.parametrize("config", [1, 3])
def test_16bit_outputs_are_the_rounded_pairs(dtype, variant, inter, config):
    th = inputs.generate(config, 0, min(inputs.size(config), 1 << 22))
    ws, wc = oracle.sincos(th, variant)
    t = torch.from_numpy(th).cuda()
    n = t.numel()
    if inter:
        o = torch.empty(2 * n, dtype=dtype, device="cuda")
        sp.sincos_pairs_dtype(t, interleaved_out=o, variant=variant)
        ob = o.view(torch.int16).cpu().numpy().view(np.uint16)
        gs, gc = ob[1::2], ob[0::2]
    else:
        s = torch.empty(n, dtype=dtype, device="cuda")
        c = torch.empty(n, dtype=dtype, device="cuda")
        sp.sincos_pairs_dtype(t, s, c, variant=variant)
        gs = s.view(torch.int16).cpu().numpy().view(np.uint16)
        gc = c.view(torch.int16).cpu().numpy().view(np.uint16)
    assert same16(gs, rn16(ws, dtype), dtype).all()
    assert same16(gc, rn16(wc, dtype), dtype).all()


@pytest.mark.parametrize("dtype", [torch.float16, torch.bfloat16])
def test_16bit_tails_and_misalignment(dtype):
    rng = np.random.default_rng(2)
    base = rng.uniform(-100, 100, 4096).astype(np.float32)
    ws, wc = oracle.sincos(base, 0)
    bt = torch.from_numpy(base).cuda()
    bs = torch.empty(4096 + 64, dtype=dtype, device="cuda")
    bc = torch.empty(4096 + 64, dtype=dtype, device="cuda")
    for n in list(range(0, 40)) + [1001, 4000]:
        for ot, oo in ((0, 0), (3, 3), (1, 0), (0, 5)):
            if ot + n > 4096:
                continue
            s, c = bs[oo:oo + n], bc[oo + 16:oo + 16 + n]
            sp.sincos_pairs_dtype(bt[ot:ot + n], s, c, variant=0)
            torch.cuda.synchronize()
            gs = s.view(torch.int16).cpu().numpy().view(np.uint16)
            gc = c.view(torch.int16).cpu().numpy().view(np.uint16)
            assert same16(gs, rn16(ws[ot:ot + n], dtype), dtype).all(), (n, ot, oo)
            assert same16(gc, rn16(wc[ot:ot + n], dtype), dtype).all(), (n, ot, oo)


def test_fp32_dtype_is_the_hot_path():
    t = torch.from_numpy(inputs.generate(2, 0, 1 << 20)).cuda()
    s1, c1 = sp.sincos(t)
    s2, c2 = torch.empty_like(t), torch.empty_like(t)
    sp.sincos_pairs_dtype(t, s2, c2)
    torch.cuda.synchronize()
    assert torch.equal(s1, s2) and torch.equal(c1, c2)


@pytest.mark.parametrize("n", [0, 1, 7, 1000, (1 << 22) + 3])
def test_adapters_round_trip(n):
    s = torch.randn(n, device="cuda")
    c = torch.randn(n, device="cuda")
    io = torch.empty(2 * n, device="cuda")
    sp.interleave(s, c, io)
    s2, c2 = torch.empty_like(s), torch.empty_like(c)
    sp.deinterleave(io, s2, c2)
    torch.cuda.synchronize()
    assert torch.equal(io[0::2], c) and torch.equal(io[1::2], s)
    assert torch.equal(s2, s) and torch.equal(c2, c)


def test_adapter_matches_interleaved_kernel_output():
    t = torch.from_numpy(inputs.generate(3, 0, 1 << 20)).cuda()
    s, c = sp.sincos(t, variant=1)
    io = torch.empty(2 * t.numel(), device="cuda")
    sp.interleave(s, c, io)
    io2 = sp.sincos(t, variant=1, interleaved=True).reshape(-1)
    torch.cuda.synchronize()
    assert torch.equal(io.view(torch.int32), io2.view(torch.int32))


@pytest.mark.parametrize("variant", [0, 1])
@pytest.mark.parametrize("dtype", ["float16", "bfloat16"])
def test_all_fp32_inputs_16bit_equal_library_rounding_of_fp32_path(variant, dtype):
    """Every one of the 2^32 fp32 inputs: the 16-bit kernel's bits equal torch's RN cast of the
    fp32 kernel's pair (whose whole-space hash equals the oracle's, test_gpu_parity), NaN
    matching NaN; split and interleaved 16-bit layouts."""
    dt = getattr(torch, dtype)
    chunk = 1 << 28
    s32 = torch.empty(chunk, dtype=torch.float32, device="cuda")
    c32 = torch.empty(chunk, dtype=torch.float32, device="cuda")
    s16 = torch.empty(chunk, dtype=dt, device="cuda")
    c16 = torch.empty(chunk, dtype=dt, device="cuda")
    i16 = torch.empty(2 * chunk, dtype=dt, device="cuda")
    bad = 0
    for u0 in range(0, 1 << 32, chunk):
        th = torch.arange(u0, u0 + chunk, dtype=torch.int64, device="cuda").to(torch.int32).view(torch.float32)
        sp.sincos_pairs(th, s32, c32, variant=variant)
        sp.sincos_pairs_dtype(th, s16, c16, variant=variant)
        sp.sincos_pairs_dtype(th, interleaved_out=i16, variant=variant)
        for got, ref in ((s16, s32), (c16, c32), (i16[1::2], s32), (i16[0::2], c32)):
            want = ref.to(dt)
            same = (got.view(torch.int16) == want.view(torch.int16)) | (torch.isnan(got) & torch.isnan(want))
            bad += int((~same).sum().item())
    assert bad == 0


@pytest.mark.parametrize("dtype", [torch.float16, torch.bfloat16])
@pytest.mark.parametrize("realign", [True, False])
def test_16bit_every_theta_offset(dtype, realign):
    """theta at every float offset 0..7 against outputs at several offsets (split with sin and
    cos sharing an offset, interleaved): the re-aligning vector body (every K = 0..7), or with
    re-alignment off the one-per-thread path; lengths around the vector boundaries and large."""
    rng = np.random.default_rng(5)
    N = 100_003
    base = rng.uniform(-300, 300, N + 16).astype(np.float32)
    with (contextlib.nullcontext() if realign else ab.knobs(realign=0)):
        for variant in (0, 1):
            ws, wc = oracle.sincos(base, variant)
            bt = torch.from_numpy(base).cuda()
            bs = torch.empty(N + 64, dtype=dtype, device="cuda")
            bc = torch.empty(N + 64, dtype=dtype, device="cuda")
            bi = torch.empty(2 * N + 64, dtype=dtype, device="cuda")
            for n in list(range(0, 20)) + [63, 64, 65, 1001, N]:
                for ot in range(8):
                    for oo in (0, 1, 6):
                        s, c = bs[oo:oo + n], bc[oo + 8:oo + 8 + n]
                        sp.sincos_pairs_dtype(bt[ot:ot + n], s, c, variant=variant)
                        io = bi[2 * oo:2 * oo + 2 * n]
                        sp.sincos_pairs_dtype(bt[ot:ot + n], interleaved_out=io, variant=variant)
                        torch.cuda.synchronize()
                        tag = (n, ot, oo, variant, realign)
                        gs = s.view(torch.int16).cpu().numpy().view(np.uint16)
                        gc = c.view(torch.int16).cpu().numpy().view(np.uint16)
                        assert same16(gs, rn16(ws[ot:ot + n], dtype), dtype).all(), tag
                        assert same16(gc, rn16(wc[ot:ot + n], dtype), dtype).all(), tag
                        gi = io.view(torch.int16).cpu().numpy().view(np.uint16)
                        assert same16(gi[1::2], rn16(ws[ot:ot + n], dtype), dtype).all(), tag
                        assert same16(gi[0::2], rn16(wc[ot:ot + n], dtype), dtype).all(), tag


@pytest.mark.parametrize("n", [1, 5, 1003, (1 << 20) + 7])
@pytest.mark.parametrize("offs", [(0, 0, 0), (1, 1, 2), (3, 0, 1), (0, 2, 0)])
def test_adapters_any_alignment(n, offs):
    """split <-> interleaved at 4-B offsets (the one-element path) and aligned (the 4-wide
    vector body with a ragged tail): exact round trip, outputs equal the inputs' layout."""
    os_, oc, oi = offs
    sb = torch.randn(n + 8, device="cuda")
    cb = torch.randn(n + 8, device="cuda")
    s, c = sb[os_:os_ + n], cb[oc:oc + n]
    ib = torch.empty(2 * n + 8, device="cuda")
    io = ib[2 * oi:2 * oi + 2 * n]
    sp.interleave(s, c, io)
    s2b, c2b = torch.empty(n + 8, device="cuda"), torch.empty(n + 8, device="cuda")
    s2, c2 = s2b[oc:oc + n], c2b[os_:os_ + n]
    sp.deinterleave(io, s2, c2)
    torch.cuda.synchronize()
    assert torch.equal(io[0::2], c) and torch.equal(io[1::2], s)
    assert torch.equal(s2, s) and torch.equal(c2, c)


@pytest.mark.parametrize("dtype", [torch.float16, torch.bfloat16])
def test_16bit_every_split_offset_pair(dtype):
    """sin and cos at every pair of element offsets 0..7 (2-B units: cos 16-, 8-, 4- or 2-B
    aligned where sin's 128-bit stores fall -- the cos[] piece stores) at two theta offsets,
    lengths around the vector boundaries; raw 16-bit values = RN of the oracle's pair; sentinel
    guard zones around both outputs."""
    SENT = 0x7E5A                       # a 16-bit NaN pattern no conversion produces
    G = 32
    N = 8 * 128 * 3 + 29
    base = inputs.generate(2, 0, N + 8)
    bt = torch.from_numpy(base).cuda()
    bs = torch.empty(2 * G + N + 16, dtype=torch.int16, device="cuda")
    bc = torch.empty_like(bs)
    bad = []
    for variant in (0, 1):
        ws, wc = oracle.sincos(base, variant)
        rs, rc = rn16(ws, dtype), rn16(wc, dtype)
        for ot in (0, 3):
            for n in list(range(0, 18)) + [63, 64, 65, 8 * 128 + 5, N]:
                for os_ in range(8):
                    for oc in range(8):
                        bs.fill_(SENT)
                        bc.fill_(SENT)
                        s = bs[G + os_:G + os_ + n].view(dtype)
                        c = bc[G + oc:G + oc + n].view(dtype)
                        sp.sincos_pairs_dtype(bt[ot:ot + n], s, c, variant=variant)
                        hs = bs.cpu().numpy().view(np.uint16)
                        hc = bc.cpu().numpy().view(np.uint16)
                        ok = (same16(hs[G + os_:G + os_ + n], rs[ot:ot + n], dtype).all() and
                              same16(hc[G + oc:G + oc + n], rc[ot:ot + n], dtype).all() and
                              (hs[:G + os_] == SENT).all() and (hs[G + os_ + n:] == SENT).all() and
                              (hc[:G + oc] == SENT).all() and (hc[G + oc + n:] == SENT).all())
                        if not ok:
                            bad.append((variant, ot, n, os_, oc))
    assert not bad, f"{len(bad)} failing (variant, theta off, n, sin off, cos off), first {bad[:8]}"
