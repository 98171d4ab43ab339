"""Guard-zone checks for out-of-bounds writes (compute-sanitizer is closed on this pool):
every entry point writes into a slice of a larger buffer pre-filled with a sentinel pattern;
everything outside the slice must still hold the sentinel afterwards.  ``pytest -m gpu``."""
import numpy as np
import pytest

import inputs

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_cs_0406049_b200 as sp  # noqa: E402

SENT = 0x7F8ABCDE          # a NaN payload no kernel produces
G = 4096                   # guard elements on each side


@pytest.fixture(scope="module", autouse=True)
def cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    yield


def check(buf, lo, hi):
    b = buf.cpu().numpy()
    assert np.all(b[:lo] == SENT) and np.all(b[hi:] == SENT), (np.flatnonzero(b[:lo] != SENT)[:5],
                                                              np.flatnonzero(b[hi:] != SENT)[:5] + hi)


SIZES = [1, 7, 8, 9, 255, 1000, 65536 + 5]
OFFS = [0, 1, 3, 5]


@pytest.mark.parametrize("n", SIZES)
@pytest.mark.parametrize("off", OFFS)
def test_pairs_split_and_interleaved(n, off):
    th = torch.from_numpy(inputs.generate(2, 0, n)).cuda()
    for v in (0, 1):
        bs = torch.full((2 * G + n + 8,), SENT, dtype=torch.int32, device="cuda")
        bc = torch.full((2 * G + n + 8,), SENT, dtype=torch.int32, device="cuda")
        s = bs[G + off:G + off + n].view(torch.float32)
        c = bc[G + off:G + off + n].view(torch.float32)
        sp.sincos_pairs(th, s, c, variant=v)
        bi = torch.full((2 * G + 2 * n + 8,), SENT, dtype=torch.int32, device="cuda")
        io = bi[G + 2 * off:G + 2 * off + 2 * n].view(torch.float32)
        sp.sincos_pairs(th, interleaved_out=io, variant=v)
        torch.cuda.synchronize()
        check(bs, G + off, G + off + n)
        check(bc, G + off, G + off + n)
        check(bi, G + 2 * off, G + 2 * off + 2 * n)


@pytest.mark.parametrize("n", SIZES)
@pytest.mark.parametrize("off", OFFS)
def test_dtype_and_method_paths(n, off):
    th = torch.from_numpy(inputs.generate(3, 0, n)).cuda()
    # 16-bit split outputs: guard in int16 units
    s16 = 0x7E5A                           # an fp16 NaN payload no kernel produces
    bs = torch.full((2 * G + n + 16,), s16, dtype=torch.int16, device="cuda")
    bc = bs.clone()
    s = bs[G + off:G + off + n].view(torch.float16)
    c = bc[G + off:G + off + n].view(torch.float16)
    sp.sincos_pairs_dtype(th, s, c, variant=1)
    torch.cuda.synchronize()
    for b in (bs, bc):
        a = b.cpu().numpy()
        assert np.all(a[:G + off] == s16) and np.all(a[G + off + n:] == s16)
    # general method
    bs = torch.full((2 * G + n + 8,), SENT, dtype=torch.int32, device="cuda")
    bc = bs.clone()
    m = sp.make_method(*sp.PAPER_METHODS[0])
    sp.sincos_pairs_method(th, m, bs[G + off:G + off + n].view(torch.float32), bc[G + off:G + off + n].view(torch.float32))
    torch.cuda.synchronize()
    check(bs, G + off, G + off + n)
    check(bc, G + off, G + off + n)


@pytest.mark.parametrize("shape", [(1, 1), (3, 8), (5, 13), (17, 1024), (64, 1000)])
def test_phase_grid_and_nudft(shape):
    nf, nt = shape
    f = torch.rand(nf, device="cuda") * 100
    t = torch.rand(nt, device="cuda")
    n = nf * nt
    bi = torch.full((2 * G + 2 * n + 8,), SENT, dtype=torch.int32, device="cuda")
    sp.phase_grid(f, t, interleaved_out=bi[G:G + 2 * n].view(torch.float32), units=sp.TURNS)
    a = torch.randn(nt, dtype=torch.complex64, device="cuda")
    bo = torch.full((2 * G + 2 * nf + 8,), SENT, dtype=torch.int32, device="cuda")
    out = bo[G:G + 2 * nf].view(torch.complex64)
    sp.nudft(f, t, a, out=out)
    torch.cuda.synchronize()
    check(bi, G, G + 2 * n)
    check(bo, G, G + 2 * nf)


@pytest.mark.parametrize("shape", [(1, 1), (3, 7), (9, 13), (33, 1001), (16, 256), (9, 131), (21, 300), (3, 4000),
                                   (21, 1), (1003, 2), (77, 3), (1000, 4), (300, 5), (129, 6), (385, 7),
                                   (128 * 9 + 3, 3), (300, 9), (129, 12), (1000, 13), (513, 14), (77, 15),
                                   (64 * 7 + 63, 10)])
@pytest.mark.parametrize("off", [0, 1, 3, 4, 6])
def test_phase_grid_split_offsets(shape, off):
    """Split phase-grid outputs at offsets (the flat kernel's head/body/tail, the ragged-row
    kernel's row ends and re-aligned t windows -- t at a float offset too -- the aligned row
    kernel, and the staged short-row kernel's regions and tail at 32-B and 16-B alignment),
    interleaved at odd and even float offsets (flat / row kernel, one pair per thread)."""
    nf, nt = shape
    f = torch.rand(nf, device="cuda") * 100
    toff = off % 5
    t = torch.rand(nt + 8, device="cuda")[toff:toff + nt]
    n = nf * nt
    bs = torch.full((2 * G + n + 8,), SENT, dtype=torch.int32, device="cuda")
    bc = bs.clone()
    sp.phase_grid(f, t, bs[G + off:G + off + n].view(torch.float32), bc[G + off:G + off + n].view(torch.float32))
    bi = torch.full((2 * G + 2 * n + 8,), SENT, dtype=torch.int32, device="cuda")
    sp.phase_grid(f, t, interleaved_out=bi[G + off:G + off + 2 * n].view(torch.float32), units=sp.TURNS)
    torch.cuda.synchronize()
    check(bs, G + off, G + off + n)
    check(bc, G + off, G + off + n)
    check(bi, G + off, G + off + 2 * n)


@pytest.mark.parametrize("n", SIZES + [8 * 128 * 3 + 5, 8 * 128 * 2 * 150 + 21])
@pytest.mark.parametrize("offs", [(0, 1, 2), (1, 0, 3), (3, 2, 0), (2, 1, 1), (0, 2, 7), (0, 3, 6)])
def test_pairs_outputs_apart(n, offs):
    """sin and cos at different offsets mod 16 B, interleaved pairs only 4-B aligned (the
    output-realigning kernel: lane 0 / last-lane edge pieces, whole blocks in between; the
    interleaved k = 3, 5, 7 instances at sizes with a partial and a full second trip)."""
    ot, os_, oc = offs
    tb = torch.from_numpy(inputs.generate(2, 0, n + 4)).cuda()
    th = tb[ot:ot + n]
    for v in (0, 1):
        bs = torch.full((2 * G + n + 8,), SENT, dtype=torch.int32, device="cuda")
        bc = torch.full((2 * G + n + 8,), SENT, dtype=torch.int32, device="cuda")
        sp.sincos_pairs(th, bs[G + os_:G + os_ + n].view(torch.float32), bc[G + oc:G + oc + n].view(torch.float32),
                        variant=v)
        bi = torch.full((2 * G + 2 * n + 8,), SENT, dtype=torch.int32, device="cuda")
        oi = 2 * os_ + 1                                  # odd: pairs 4-B aligned only
        sp.sincos_pairs(th, interleaved_out=bi[G + oi:G + oi + 2 * n].view(torch.float32), variant=v)
        torch.cuda.synchronize()
        check(bs, G + os_, G + os_ + n)
        check(bc, G + oc, G + oc + n)
        check(bi, G + oi, G + oi + 2 * n)


@pytest.mark.parametrize("n", SIZES + [8 * 40_000 + 3])
@pytest.mark.parametrize("off", [0, 1, 2, 4, 8])
def test_layout_adapters(n, off):
    """sincos_interleave / sincos_deinterleave (the 256-bit form when all three buffers are 32-B
    aligned -- off 0, 8 -- else the 128-bit or scalar forms): no write outside the outputs, and
    the round trip is exact."""
    s = torch.rand(n, device="cuda")
    c = torch.rand(n, device="cuda")
    bi = torch.full((2 * G + 2 * n + 16,), SENT, dtype=torch.int32, device="cuda")
    io = bi[G + 2 * off:G + 2 * off + 2 * n].view(torch.float32)
    sp.interleave(s, c, io)
    bs = torch.full((2 * G + n + 16,), SENT, dtype=torch.int32, device="cuda")
    bc = bs.clone()
    s2 = bs[G + off:G + off + n].view(torch.float32)
    c2 = bc[G + off:G + off + n].view(torch.float32)
    sp.deinterleave(io, s2, c2)
    torch.cuda.synchronize()
    check(bi, G + 2 * off, G + 2 * off + 2 * n)
    check(bs, G + off, G + off + n)
    check(bc, G + off, G + off + n)
    assert torch.equal(s2, s) and torch.equal(c2, c)
    assert torch.equal(io.view(n, 2)[:, 0], c) and torch.equal(io.view(n, 2)[:, 1], s)
