"""Every split (sin, cos) pointer layout through the product dispatch, compared by raw bits
with the oracle and guard-zone checked (``pytest -m gpu``).

The layout picks the kernel form: shared alignment -> the vector kernel;
theta off outputs that share their offset mod 32 B -> KB3b; sin and cos apart with one of them
at theta's frame -> KB3c re-aligning that one stream; both apart from theta's frame and from each
other -> the hybrid KB3c form (theta re-aligned onto one output's frame, the other stream
re-aligned).  All 64 (sin, cos) offsets 0..7 floats at three theta offsets, lengths around the
vector, warp and block boundaries, both variants, outputs inside sentinel-filled buffers."""
import numpy as np
import pytest

import inputs
import oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_cs_0406049_b200 as sp  # noqa: E402

SENT = 0x7F8ABCDE          # a NaN payload no kernel produces
G = 64                     # guard elements on each side (in floats)
NMAX = 8 * 128 * 3 * 2 + 77
LENGTHS = list(range(0, 18)) + [23, 24, 25, 31, 255, 256, 257, 8 * 32 + 9, 8 * 32 * 4 - 1, 8 * 128 + 15,
                                8 * 128 * 3 + 5, NMAX]


@pytest.fixture(scope="module")
def data():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    base = inputs.generate(2, 0, NMAX + 8)
    want = {}
    for v in (oracle.VARIANT_N, oracle.VARIANT_A):
        s, c = oracle.sincos(base, v)
        want[v] = (torch.from_numpy(s.view(np.int32)).cuda(), torch.from_numpy(c.view(np.int32)).cuda())
    return torch.from_numpy(base).cuda(), want


@pytest.mark.parametrize("variant", [oracle.VARIANT_N, oracle.VARIANT_A])
@pytest.mark.parametrize("ot", [0, 3, 6])
def test_every_split_layout(data, variant, ot):
    tb, want = data
    ws, wc = want[variant]
    bs = torch.empty(2 * G + NMAX + 8, dtype=torch.int32, device="cuda")
    bc = torch.empty_like(bs)
    bad = []
    for os_ in range(8):
        for oc in range(8):
            for n in LENGTHS:
                bs.fill_(SENT)
                bc.fill_(SENT)
                s = bs[G + os_:G + os_ + n].view(torch.float32)
                c = bc[G + oc:G + oc + n].view(torch.float32)
                sp.sincos_pairs(tb[ot:ot + n], s, c, variant=variant)
                ok = (torch.equal(bs[G + os_:G + os_ + n], ws[ot:ot + n]) and
                      torch.equal(bc[G + oc:G + oc + n], wc[ot:ot + n]) and
                      bool((bs[:G + os_] == SENT).all()) and bool((bs[G + os_ + n:] == SENT).all()) and
                      bool((bc[:G + oc] == SENT).all()) and bool((bc[G + oc + n:] == SENT).all()))
                if not ok:
                    bad.append((os_, oc, n))
    assert not bad, f"theta+{ot} variant {variant}: {len(bad)} failing (sin off, cos off, n), first {bad[:8]}"


@pytest.mark.parametrize("variant", [oracle.VARIANT_N, oracle.VARIANT_A])
def test_every_split_layout_grid_stride(variant):
    """The same 64 (sin, cos) offset pairs on the A/B build with a grid of one block per SM, so
    every warp makes several grid-stride trips (the hybrid's warp-edge blocks meet across trips),
    at two theta offsets and a length with a ragged tail."""
    from paper_cs_0406049_b200 import ab
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    n = 400_003
    base = inputs.generate(3, 0, n + 8)
    s_, c_ = oracle.sincos(base, variant)
    ws = torch.from_numpy(s_.view(np.int32)).cuda()
    wc = torch.from_numpy(c_.view(np.int32)).cuda()
    tb = torch.from_numpy(base).cuda()
    bs = torch.empty(2 * G + n + 8, dtype=torch.int32, device="cuda")
    bc = torch.empty_like(bs)
    bad = []
    with ab.knobs(blocks_per_sm=1):
        for ot in (0, 5):
            for os_ in range(8):
                for oc in range(8):
                    bs.fill_(SENT)
                    bc.fill_(SENT)
                    sp.sincos_pairs(tb[ot:ot + n], bs[G + os_:G + os_ + n].view(torch.float32),
                                    bc[G + oc:G + oc + n].view(torch.float32), variant=variant)
                    ok = (torch.equal(bs[G + os_:G + os_ + n], ws[ot:ot + n]) and
                          torch.equal(bc[G + oc:G + oc + n], wc[ot:ot + n]) and
                          bool((bs[:G + os_] == SENT).all()) and bool((bs[G + os_ + n:] == SENT).all()) and
                          bool((bc[:G + oc] == SENT).all()) and bool((bc[G + oc + n:] == SENT).all()))
                    if not ok:
                        bad.append((ot, os_, oc))
    assert not bad, f"variant {variant}: {len(bad)} failing (theta off, sin off, cos off), first {bad[:8]}"
