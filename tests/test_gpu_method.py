"""GPU parity of NEXT(3), sincos_pairs_method (caller-supplied series / doublings / fix),
against the oracle's general method: bit-exact by value.  ``pytest -m gpu``."""
import contextlib
import numpy as np
import pytest

import inputs
import oracle
from helpers import assert_parity
from paper_cs_0406049_b200 import coeff_fit as cf

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_cs_0406049_b200 as sp  # noqa: E402
from paper_cs_0406049_b200 import ab  # noqa: E402  (A/B build)

OFIX = {sp.FIX_LINEAR: oracle.FIX_LINEAR_PENULTIMATE, sp.FIX_RECIPROCAL: oracle.FIX_RECIPROCAL,
        sp.FIX_NONE: oracle.FIX_NONE}


@pytest.fixture(scope="module", autouse=True)
def cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    yield


def methods():
    out = []
    for v in (sp.NORMALIZED, sp.RENORMALIZED):
        ss, cc, n, fix = sp.PAPER_METHODS[v]
        out.append(("paper" + "NA"[v], ss, cc, n, fix))
    for n, ds, dc, kind in [(2, 4, 3, "n"), (2, 3, 3, "a"), (3, 3, 3, "a"), (1, 5, 5, "a"), (2, 5, 4, "n"),
                            (4, 3, 2, "a"), (1, 8, 8, "n")]:
        f = cf.fit_normalized(n, ds, dc, weight="relative") if kind == "n" else cf.fit_angle(n, ds, dc)
        ss, cc = f.fp32()
        out.append((f"fit{kind}{n}_{ds}{dc}", list(ss), list(cc), n, sp.FIX_LINEAR if kind == "n" else sp.FIX_RECIPROCAL))
    out.append(("nofix0", [1.5707964, -0.6459], [], 0, sp.FIX_NONE))
    out.append(("nofix2", list(sp.PAPER_METHODS[0][0]), list(sp.PAPER_METHODS[0][1]), 2, sp.FIX_NONE))
    return out


def omethod(ss, cc, n, fix):
    return oracle.make_method(np.float32(ss), np.float32(cc), n, OFIX[fix])


@pytest.mark.parametrize("name,ss,cc,n,fix", methods(), ids=[m[0] for m in methods()])
@pytest.mark.parametrize("inter", [False, True])
def test_method_parity(name, ss, cc, n, fix, inter):
    th = np.concatenate([inputs.generate(2, 0, (1 << 20) + 3), inputs.generate(3, 0, 1 << 18)])
    t = torch.from_numpy(th).cuda()
    m = sp.make_method(ss, cc, n, fix)
    if inter:
        o = torch.empty(2 * t.numel(), device="cuda")
        sp.sincos_pairs_method(t, m, interleaved_out=o)
        o = o.cpu().numpy()
        gs, gc = o[1::2], o[0::2]
    else:
        s, c = torch.empty_like(t), torch.empty_like(t)
        sp.sincos_pairs_method(t, m, s, c)
        gs, gc = s.cpu().numpy(), c.cpu().numpy()
    ws, wc = oracle.method_sincos(th, omethod(ss, cc, n, fix))
    assert_parity(gs, gc, ws, wc, name)


@pytest.mark.parametrize("variant", [sp.NORMALIZED, sp.RENORMALIZED])
def test_paper_tables_equal_the_hot_path(variant):
    """The paper's tables through the general kernel are bit-identical to sincos_pairs."""
    t = torch.from_numpy(inputs.generate(2, 0, 1 << 24)).cuda()
    s1, c1 = sp.sincos(t, variant=variant)
    s2, c2 = torch.empty_like(t), torch.empty_like(t)
    sp.sincos_pairs_method(t, sp.make_method(*sp.PAPER_METHODS[variant]), s2, c2)
    torch.cuda.synchronize()
    assert torch.equal(s1, s2) and torch.equal(c1, c2)


def test_method_tails_and_misalignment():
    rng = np.random.default_rng(3)
    base = rng.uniform(-100, 100, 4096).astype(np.float32)
    f = cf.fit_angle(3, 3, 3)
    ss, cc = f.fp32()
    m = sp.make_method(list(ss), list(cc), 3, sp.FIX_RECIPROCAL)
    ws, wc = oracle.method_sincos(base, omethod(list(ss), list(cc), 3, sp.FIX_RECIPROCAL))
    bt = torch.from_numpy(base).cuda()
    bs = torch.empty(4096 + 64, device="cuda")
    bc = torch.empty(4096 + 64, device="cuda")
    for n in list(range(0, 40)) + [1000, 4000]:
        for ot, oo in ((0, 0), (3, 3), (1, 0)):
            if ot + n > 4096:
                continue
            s, c = bs[oo:oo + n], bc[oo + 8:oo + 8 + n]
            sp.sincos_pairs_method(bt[ot:ot + n], m, s, c)
            torch.cuda.synchronize()
            assert_parity(s.cpu().numpy(), c.cpu().numpy(), ws[ot:ot + n], wc[ot:ot + n], f"n={n}")


def test_method_validation():
    t = torch.zeros(16, device="cuda")
    s, c = torch.empty_like(t), torch.empty_like(t)
    for bad in (sp.make_method([], [], 2, 0), sp.make_method([1.0], [], 0, sp.FIX_LINEAR),
                sp.make_method([1.0] * 9 if False else [1.0], [], 9, 0)):
        with pytest.raises(sp.SincosError):
            sp.sincos_pairs_method(t, bad, s, c)
    with pytest.raises(sp.SincosError):
        sp.sincos_pairs_method(t, sp.make_method([1.0], [], 2, 0), t, c)     # in-place not supported


@pytest.mark.parametrize("realign", [True, False])
def test_method_every_theta_offset(realign):
    """The general-method kernel with theta at every float offset 0..7 against split outputs
    (sin and cos at one offset) and interleaved outputs at 8-B and 4-B offsets: the re-aligning
    vector body for every K, or one element per thread; bit-exact vs the oracle's method."""
    rng = np.random.default_rng(4)
    N = 100_003
    base = rng.uniform(-300, 300, N + 16).astype(np.float32)
    f = cf.fit_angle(1, 3, 2)
    ss, cc = f.fp32()
    m = sp.make_method(list(ss), list(cc), 1, sp.FIX_RECIPROCAL)
    ws, wc = oracle.method_sincos(base, omethod(list(ss), list(cc), 1, sp.FIX_RECIPROCAL))
    bt = torch.from_numpy(base).cuda()
    bs = torch.empty(N + 64, device="cuda")
    bc = torch.empty(N + 64, device="cuda")
    bi = torch.empty(2 * N + 64, device="cuda")
    with (contextlib.nullcontext() if realign else ab.knobs(realign=0)):
        for n in list(range(0, 20)) + [63, 64, 65, 1001, N]:
            for ot in range(8):
                for oo in (0, 1, 6):
                    s, c = bs[oo:oo + n], bc[oo + 8:oo + 8 + n]
                    sp.sincos_pairs_method(bt[ot:ot + n], m, s, c)
                    io = bi[oo:oo + 2 * n]                    # oo odd: only 4-B aligned pairs
                    sp.sincos_pairs_method(bt[ot:ot + n], m, interleaved_out=io)
                    torch.cuda.synchronize()
                    tag = f"n={n} ot={ot} oo={oo} realign={realign}"
                    assert_parity(s.cpu().numpy(), c.cpu().numpy(), ws[ot:ot + n], wc[ot:ot + n], tag)
                    iv = io.cpu().numpy()
                    assert_parity(iv[1::2], iv[0::2], ws[ot:ot + n], wc[ot:ot + n], "inter " + tag)


@pytest.mark.parametrize("fix", [sp.FIX_LINEAR, sp.FIX_RECIPROCAL])
def test_method_every_split_offset_pair(fix):
    """The general-method kernel with sin and cos at every pair of float offsets 0..7 (cos off
    sin's 32-B frame: re-aligned by warp shuffles) at two theta offsets, lengths around the
    vector / warp boundaries; raw bits equal the oracle's method, sentinel guard zones."""
    SENT = 0x7F8ABCDE
    G = 64
    N = 8 * 128 * 3 + 77
    base = inputs.generate(2, 0, N + 8)
    f = cf.fit_angle(1, 3, 2)
    ss, cc = f.fp32()
    m = sp.make_method(list(ss), list(cc), 1, fix)
    ws, wc = oracle.method_sincos(base, omethod(list(ss), list(cc), 1, fix))
    ws_i = torch.from_numpy(np.ascontiguousarray(ws).view(np.int32)).cuda()
    wc_i = torch.from_numpy(np.ascontiguousarray(wc).view(np.int32)).cuda()
    bt = torch.from_numpy(base).cuda()
    bs = torch.empty(2 * G + N + 8, dtype=torch.int32, device="cuda")
    bc = torch.empty_like(bs)
    bad = []
    for ot in (0, 3):
        for n in list(range(0, 18)) + [63, 64, 65, 8 * 32 + 5, 8 * 128 + 9, N]:
            for os_ in range(8):
                for oc in range(8):
                    bs.fill_(SENT)
                    bc.fill_(SENT)
                    sp.sincos_pairs_method(bt[ot:ot + n], m, bs[G + os_:G + os_ + n].view(torch.float32),
                                           bc[G + oc:G + oc + n].view(torch.float32))
                    ok = (torch.equal(bs[G + os_:G + os_ + n], ws_i[ot:ot + n]) and
                          torch.equal(bc[G + oc:G + oc + n], wc_i[ot:ot + n]) and
                          bool((bs[:G + os_] == SENT).all()) and bool((bs[G + os_ + n:] == SENT).all()) and
                          bool((bc[:G + oc] == SENT).all()) and bool((bc[G + oc + n:] == SENT).all()))
                    if not ok:
                        bad.append((ot, n, os_, oc))
    assert not bad, f"{len(bad)} failing (theta off, n, sin off, cos off), first {bad[:8]}"
