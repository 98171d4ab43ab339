"""Seeded random sweep of the C ABI's pair paths against the oracle (``pytest -m gpu``).

Each case draws a length (0 .. ~300k, biased to the small and ragged), element offsets of
theta and of each output buffer (so every kernel form is reached: the 256-bit and 128-bit
vector bodies, the re-aligning kernels, one element per thread), a layout (split /
interleaved), a variant, an entry point (sincos_pairs, sincos_pairs_dtype fp32,
sincos_pairs_method with the paper's table, sincos_phase_grid with f = [1] in radians -- all
of which must return the method's pairs), a launch configuration and an input distribution
(the five BASELINE config generators, raw bit patterns).  Bar: bit-exact by value vs the
oracle on the same inputs."""
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

CASES = 800


@pytest.fixture(scope="module", autouse=True)
def cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    yield


def draw_theta(rng, n):
    kind = rng.integers(0, 7)
    if kind < 5:
        return inputs.generate(int(kind) + 1, int(rng.integers(0, 1 << 20)), n)
    if kind == 5:
        return rng.integers(0, 1 << 32, n, dtype=np.uint64).astype(np.uint32).view(np.float32)
    return rng.uniform(-1e6, 1e6, n).astype(np.float32)


@pytest.mark.parametrize("block", range(8))
def test_fuzz_pairs(block):
    rng = np.random.default_rng(1000 + block)
    for case in range(CASES // 8):
        r = rng.random()
        n = int(rng.integers(0, 40)) if r < 0.3 else int(rng.integers(40, 5000)) if r < 0.8 \
            else int(rng.integers(5000, 300_000))
        variant = int(rng.integers(0, 2))
        inter = bool(rng.integers(0, 2))
        entry = ["pairs", "dtype32", "method", "phase", "phase2d"][int(rng.integers(0, 5))]
        if entry == "phase2d":                           # an nf x nt grid: theta_ij = RN(f_i t_j)
            if rng.random() < 0.5:                        # many short rows (tiny / staged / short-row kernels)
                nt2 = int(rng.integers(1, 16))
                nf2 = max(1, n // nt2)
            else:
                nf2 = int(rng.integers(1, 24))
                nt2 = max(1, n // nf2)
            f2 = rng.uniform(-50, 50, nf2).astype(np.float32)
            t2 = draw_theta(rng, nt2 + 8)
            toff2 = int(rng.integers(0, 8))
            t2 = t2[toff2:toff2 + nt2]
            n = nf2 * nt2
            with np.errstate(over="ignore", invalid="ignore"):   # inf / NaN products are inputs too
                th = (f2[:, None] * t2[None, :]).astype(np.float32).ravel()   # IEEE fp32 products
        else:
            th = draw_theta(rng, n)
        ot, os_, oc = (int(x) for x in rng.integers(0, 8, 3))
        if rng.random() < 0.5:
            oc = os_                                     # sin and cos at one offset (common)
        # half the cases on the product library, half on the A/B build with a random launch
        # shape and, 15% of the time, re-alignment off (one element per thread)
        cfg = [(128, 0, 8, 1, 0), (256, 0, 8, 2, 0), (512, 4, 4, 1, 1), (128, 1, 8, 4, 0)][int(rng.integers(0, 4))]
        realign = int(rng.random() < 0.85)
        use_ab = rng.random() < 0.5
        if not use_ab:
            cfg, realign = "product", 1
        ctx = ab.knobs(launch=cfg, realign=realign) if use_ab else contextlib.nullcontext()
        ctx.__enter__()
        tbuf = torch.empty(n + 16, dtype=torch.float32, device="cuda")
        tbuf[ot:ot + n].copy_(torch.from_numpy(th))
        t = tbuf[ot:ot + n]
        if inter:
            ibuf = torch.empty(2 * n + 16, dtype=torch.float32, device="cuda")
            io = ibuf[os_:os_ + 2 * n]                   # odd os_: pairs only 4-B aligned
            outs = {"interleaved_out": io}
        else:
            sbuf = torch.empty(n + 16, dtype=torch.float32, device="cuda")
            cbuf = torch.empty(n + 16, dtype=torch.float32, device="cuda")
            outs = {"sin_out": sbuf[os_:os_ + n], "cos_out": cbuf[oc:oc + n]}
        if entry == "pairs":
            sp.sincos_pairs(t, variant=variant, **outs)
        elif entry == "dtype32":
            sp.sincos_pairs_dtype(t, variant=variant, **outs)
        elif entry == "method":
            sp.sincos_pairs_method(t, sp.make_method(*sp.PAPER_METHODS[variant]), **outs)
        elif entry == "phase":
            one = torch.ones(1, dtype=torch.float32, device="cuda")
            sp.phase_grid(one, t, units=sp.RADIANS, variant=variant, **outs)
        else:
            tb2 = torch.empty(nt2 + 8, dtype=torch.float32, device="cuda")
            tb2[toff2:toff2 + nt2].copy_(torch.from_numpy(t2))
            sp.phase_grid(torch.from_numpy(f2).cuda(), tb2[toff2:toff2 + nt2], units=sp.RADIANS, variant=variant,
                          **outs)
        torch.cuda.synchronize()
        ctx.__exit__(None, None, None)
        if inter:
            v = outs["interleaved_out"].cpu().numpy()
            gs, gc = v[1::2], v[0::2]
        else:
            gs, gc = outs["sin_out"].cpu().numpy(), outs["cos_out"].cpu().numpy()
        ws, wc = oracle.sincos(th, variant)
        assert_parity(gs, gc, ws, wc, f"case {block}/{case}: n={n} entry={entry} inter={inter} v={variant} "
                                      f"offs={ot},{os_},{oc} cfg={cfg} realign={realign}")
