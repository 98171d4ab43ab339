"""Full-array parity at BASELINE.json's largest sizes, every element (``pytest -m gpu``).

north_star: "GPU output matching the oracle ... on all five configs".  C1-C3 are compared in
full in test_gpu_parity.py; here C4 (configs[3], 2^30 NUFFT phases) and C5 (configs[4], 2^32
normal angles, 16 GiB in / 32 GiB out) run on one GPU at full size, in the launch
configuration bench.py times (one launch over the whole array), both variants, both output
layouts, and every element is compared with the oracle on the regenerated inputs -- chunk by
chunk: the host regenerates a chunk of theta (the shared generator), runs the threaded C
oracle on it, copies its pairs to the device and compares there.

The comparison is of BIT PATTERNS (only NaN payloads are excused, G8): a sign-of-zero
difference (the kernel's RN product vs Fig. 1's vec_madd(a, b, 0.0) = fmaf(a, b, +0)) would
fail here, and the same raw comparison runs over all 2^32 fp32 bit patterns, where every
signed zero, subnormal and non-finite input occurs.  Runtime (one B200 box, 16 host threads):
about a minute in all, dominated by the host generator and oracle.
"""
import time

import numpy as np
import pytest

import inputs
from helpers import oracle_threaded

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_cs_0406049_b200 as sp  # noqa: E402

CHUNK = 1 << 27


@pytest.fixture(scope="module", autouse=True)
def cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    yield
    torch.cuda.empty_cache()


def gen_to_device(config, n):
    dev = torch.empty(n, dtype=torch.float32, device="cuda")
    host = torch.empty(min(CHUNK, n), dtype=torch.float32).pin_memory()
    for off in range(0, n, CHUNK):
        m = min(CHUNK, n - off)
        inputs.generate(config, off, m, out=host.numpy()[:m])
        dev[off:off + m].copy_(host[:m])
    return dev


def bit_mismatches(got, want):
    """Positions where the float32 tensors differ in bit pattern (NaN matching any NaN)."""
    same = (got.view(torch.int32) == want.view(torch.int32)) | (torch.isnan(got) & torch.isnan(want))
    return torch.nonzero(~same).flatten()


def full_compare(config, variant):
    """Every element of config `config`, one variant, split and interleaved outputs."""
    n = inputs.size(config)
    t0 = time.perf_counter()
    th = gen_to_device(config, n)
    s = torch.empty(n, dtype=torch.float32, device="cuda")
    c = torch.empty(n, dtype=torch.float32, device="cuda")
    io = torch.empty(2 * n, dtype=torch.float32, device="cuda")
    before = sp.launch_count()
    sp.sincos_pairs(th, s, c, variant=variant)                  # one launch each, whole array
    sp.sincos_pairs(th, interleaved_out=io, variant=variant)
    torch.cuda.synchronize()
    assert sp.launch_count() - before == 2
    pairs = io.view(n, 2)
    checked = 0
    for off in range(0, n, CHUNK):
        m = min(CHUNK, n - off)
        th_h = inputs.generate(config, off, m)                     # regenerated on the host
        ws, wc = oracle_threaded(th_h, variant)
        wsd, wcd = torch.from_numpy(ws).cuda(), torch.from_numpy(wc).cuda()
        for name, got_s, got_c in (("split", s[off:off + m], c[off:off + m]),
                                   ("interleaved", pairs[off:off + m, 1], pairs[off:off + m, 0])):
            for comp, got, want in (("sin", got_s, wsd), ("cos", got_c, wcd)):
                bad = bit_mismatches(got, want)
                if bad.numel():
                    i = int(bad[0])
                    raise AssertionError(
                        f"config {config} variant {variant} {name} {comp}: {bad.numel()} bit mismatches in chunk "
                        f"at {off}; first at {off + i}: theta {th_h[i]!r} got {float(got[i])!r} "
                        f"(0x{int(got.view(torch.int32)[i]) & 0xFFFFFFFF:08X}) want {float(want[i])!r} "
                        f"(0x{int(want.view(torch.int32)[i]) & 0xFFFFFFFF:08X})")
        checked += m
    assert checked == n
    del th, s, c, io
    torch.cuda.empty_cache()
    return time.perf_counter() - t0


@pytest.mark.parametrize("variant", [0, 1])
def test_c4_full(variant):
    """BASELINE configs[3]: 2^30 NUFFT phases 2 pi f_i t_j (seed 3), every element, split and
    interleaved, bit for bit."""
    dt = full_compare(4, variant)
    print(f"C4 variant {variant}: 2^30 elements x 2 layouts in {dt:.1f} s")


@pytest.mark.parametrize("variant", [0, 1])
def test_c5_full(variant):
    """BASELINE configs[4]: 2^32 N(0, 100^2) (seed 4), 64-bit indexing past 2^31 and 2^32-1,
    every element, split and interleaved, bit for bit."""
    dt = full_compare(5, variant)
    print(f"C5 variant {variant}: 2^32 elements x 2 layouts in {dt:.1f} s")


@pytest.mark.parametrize("variant", [0, 1])
def test_all_fp32_bit_patterns_raw_bits(variant):
    """Every one of the 2^32 fp32 inputs (theta_i = bits(i)): the kernel's output BITS equal the
    oracle's, split and interleaved -- signed zeros included (the whole-space hash tests
    canonicalise +-0; this one does not), NaN payloads excused."""
    dt = full_compare(0, variant)
    print(f"all 2^32 bit patterns variant {variant}: x 2 layouts in {dt:.1f} s")


def c4_axes(turns):
    """BASELINE configs[3] axes (2^15 f x 2^15 jittered t); in radians the row factor is fl32(2 pi f)."""
    nf = nt = 1 << 15
    f = np.array([512.0 * inputs.urand(3, 0, i) for i in range(nf)])
    t = np.array([(j + inputs.urand(3, 1, j)) * 2.0 ** -15 for j in range(nt)])
    if not turns:
        f = 2 * np.pi * f
    return f.astype(np.float32), t.astype(np.float32)


def oracle_grid_rows(f, t, units, variant, rows):
    """oracle.phase_grid over blocks of rows on all host threads (per-pair numerics unchanged)."""
    import os
    from concurrent.futures import ThreadPoolExecutor

    import oracle
    spans = [(i, min(i + rows // 64, rows)) for i in range(0, rows, max(1, rows // 64))]
    with ThreadPoolExecutor(os.cpu_count() or 1) as ex:
        parts = list(ex.map(lambda ab: oracle.phase_grid(f[ab[0]:ab[1]], t, units, variant), spans))
    return np.concatenate([p[0] for p in parts]).ravel(), np.concatenate([p[1] for p in parts]).ravel()


@pytest.mark.parametrize("units", [0, 1])
@pytest.mark.parametrize("variant", [0, 1])
def test_c4_phase_grid_full(units, variant):
    """NEXT(1) at BASELINE configs[3]'s full shape: the 2^15 x 2^15 phase grid formed in the kernel
    (2^30 pairs), split and interleaved, every element, raw bits, against the oracle's pairs of
    RN(f_i t_j) -- 4096 rows at a time."""
    nf = nt = 1 << 15
    f, t = c4_axes(units == 1)
    fd, td = torch.from_numpy(f).cuda(), torch.from_numpy(t).cuda()
    n = nf * nt
    s = torch.empty(n, device="cuda")
    c = torch.empty(n, device="cuda")
    io = torch.empty(2 * n, device="cuda")
    sp.phase_grid(fd, td, s, c, units=units, variant=variant)
    sp.phase_grid(fd, td, interleaved_out=io, units=units, variant=variant)
    torch.cuda.synchronize()
    pairs = io.view(n, 2)
    R = 4096
    for r0 in range(0, nf, R):
        ws, wc = oracle_grid_rows(f[r0:r0 + R], t, units, variant, R)
        wsd, wcd = torch.from_numpy(ws).cuda(), torch.from_numpy(wc).cuda()
        lo, hi = r0 * nt, (r0 + R) * nt
        for name, gs, gc in (("split", s[lo:hi], c[lo:hi]), ("interleaved", pairs[lo:hi, 1], pairs[lo:hi, 0])):
            for comp, got, want in (("sin", gs, wsd), ("cos", gc, wcd)):
                bad = bit_mismatches(got, want)
                assert bad.numel() == 0, f"{name} {comp}: {bad.numel()} mismatches from row {r0}, first {int(bad[0])}"
    del s, c, io
    torch.cuda.empty_cache()


@pytest.mark.parametrize("inter", [False, True])
def test_beyond_2_pow_32_elements(inter):
    """64-bit indexing past C5: n = 2^33 + 13 angles (split: 96 GiB resident; interleaved: 96 GiB)
    in one launch.  theta is one 2^28-element block of C2 tiled 32 times (+13), so element i is
    block[i mod 2^28]: every tile's outputs must equal the first tile's bit for bit, and sampled
    elements -- both ends, around 2^31, 2^32 and 2^33 -- equal the oracle."""
    import oracle
    B = 1 << 28
    n = (1 << 33) + 13
    free, _ = torch.cuda.mem_get_info()
    if free < 12 * n + (8 << 30):
        pytest.skip(f"needs {12 * n / 2**30:.0f} GiB free")
    block = inputs.generate(2, 0, B)
    th = torch.empty(n, dtype=torch.float32, device="cuda")
    bd = torch.from_numpy(block).cuda()
    for k in range(0, n, B):
        m = min(B, n - k)
        th[k:k + m].copy_(bd[:m])
    del bd
    if inter:
        io = torch.empty(2 * n, dtype=torch.float32, device="cuda")
        sp.sincos_pairs(th, interleaved_out=io, variant=1)
        pv = io.view(n, 2)
        s, c = pv[:, 1], pv[:, 0]
    else:
        s = torch.empty(n, dtype=torch.float32, device="cuda")
        c = torch.empty(n, dtype=torch.float32, device="cuda")
        sp.sincos_pairs(th, s, c, variant=1)
    torch.cuda.synchronize()
    del th
    s0, c0 = s[:B].clone(), c[:B].clone()
    for k in range(B, n, B):
        m = min(B, n - k)
        assert bit_mismatches(s[k:k + m], s0[:m]).numel() == 0, f"tile at {k}"
        assert bit_mismatches(c[k:k + m], c0[:m]).numel() == 0, f"tile at {k}"
    idx = np.unique(np.concatenate([np.arange(0, 64), np.arange(n - 64, n),
                                    np.arange((1 << 31) - 32, (1 << 31) + 32),
                                    np.arange((1 << 32) - 32, (1 << 32) + 32),
                                    np.arange((1 << 33) - 32, (1 << 33) + 13)])).astype(np.int64)
    it = torch.from_numpy(idx).cuda()
    ws, wc = oracle.sincos(block[idx % B], 1)
    gs, gc = s[it].cpu().numpy(), c[it].cpu().numpy()
    assert np.array_equal(gs.view(np.uint32), ws.view(np.uint32))       # (C2 has no NaN)
    assert np.array_equal(gc.view(np.uint32), wc.view(np.uint32))
    del s, c, s0, c0
    torch.cuda.empty_cache()
