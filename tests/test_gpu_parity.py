"""GPU parity: the CUDA path (through the C ABI) against the oracle, element by element
(SURVEY 4 tier T2).  All tests need a B200: ``pytest -m gpu``.

Bar: bit-exact by value (signed zeros and NaN payloads aside; reading G15 -- the
algorithm fixes one bit pattern per input), which implies the north_star bound
|delta| <= 4 ulp of 1.0 per component (ULP4 in helpers.py), also asserted."""
import contextlib
import math
import os

import numpy as np
import pytest

import inputs
import oracle
from helpers import assert_parity, oracle_threaded

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_cs_0406049_b200 as sp  # noqa: E402
from paper_cs_0406049_b200 import ab  # noqa: E402  (A/B build: the alternative kernel forms)

VARIANTS = [oracle.VARIANT_N, oracle.VARIANT_A]   # same numbering as sp.NORMALIZED / sp.RENORMALIZED


@pytest.fixture(scope="module", autouse=True)
def cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.init()
    yield


def run(theta_np, variant, inter=False):
    t = torch.from_numpy(np.ascontiguousarray(theta_np, dtype=np.float32)).cuda()
    if inter:
        o = torch.empty(2 * t.numel(), dtype=torch.float32, device="cuda")
        sp.sincos_pairs(t, interleaved_out=o, variant=variant)
        torch.cuda.synchronize()
        o = o.cpu().numpy()
        return o[1::2].copy(), o[0::2].copy()
    s, c = torch.empty_like(t), torch.empty_like(t)
    sp.sincos_pairs(t, s, c, variant=variant)
    torch.cuda.synchronize()
    return s.cpu().numpy(), c.cpu().numpy()


# ---- configs C1 and C3 in full, C2 in full at bench size -------------------------------

@pytest.mark.parametrize("variant", VARIANTS)
@pytest.mark.parametrize("inter", [False, True])
def test_c1_full(variant, inter):
    """BASELINE configs[0]: 2^20 U[-pi, pi), seed 0 -- every element vs the oracle, and the
    error vs long double never exceeds the oracle's own (BJ:5)."""
    th = inputs.generate(1)
    s, c = run(th, variant, inter)
    os_, oc = oracle.sincos(th, variant)
    assert_parity(s, c, os_, oc, "C1")
    g = oracle.error_stats(th, s, c, oracle.REF_LONGDOUBLE)
    o = oracle.error_stats(th, os_, oc, oracle.REF_LONGDOUBLE)
    assert g.max_comb <= o.max_comb and g.count == th.size
    assert g.max_comb <= 1.25 * (4.8e-7 if variant == 0 else 3.8e-7)


@pytest.mark.parametrize("variant", VARIANTS)
def test_c3_edge_set_full(variant):
    """BASELINE configs[2]: 2^24 edge/stress set (multiples of pi/2 and pi, +-64 ulp around
    (2n+1)pi, signed zeros, subnormals, log-uniform 1e-30..2^20), interleaved output."""
    th = inputs.generate(3)
    s, c = run(th, variant, inter=True)
    os_, oc = oracle_threaded(th, variant)
    assert_parity(s, c, os_, oc, "C3")
    # signed zeros and subnormals: sin(+-0) == 0, cos == 1; subnormal sine is gradual
    z = th == 0
    assert np.all(s[z] == 0) and np.all(c[z] == 1)
    sub = (th != 0) & (np.abs(th) < np.float32(2.0 ** -126))
    assert np.all(c[sub] == 1) and np.count_nonzero(s[sub]) > 0.9 * np.count_nonzero(sub)


@pytest.mark.parametrize("variant", VARIANTS)
def test_c2_full_size(variant):
    """BASELINE configs[1]: 2^28 U[-1e4, 1e4], seed 1, split, every element, in the launch
    configuration bench.py times."""
    th = inputs.generate(2)
    s, c = run(th, variant)
    os_, oc = oracle_threaded(th, variant)
    assert_parity(s, c, os_, oc, "C2")


def sampled_indices(n, m=1 << 20, seed=0):
    rng = np.random.default_rng(seed)
    idx = np.concatenate([np.arange(0, 4096), np.arange(n - 4096, n), rng.integers(0, n, m)])
    return np.unique(idx).astype(np.int64)


def gen_to_device(config, n, chunk=1 << 28):
    dev = torch.empty(n, dtype=torch.float32, device="cuda")
    host = torch.empty(min(chunk, n), dtype=torch.float32).pin_memory()
    for off in range(0, n, chunk):
        m = min(chunk, n - off)
        inputs.generate(config, off, m, out=host.numpy()[:m])
        dev[off:off + m].copy_(host[:m])
    return dev


def test_c4_full_size_sampled():
    """BASELINE configs[3]: 2^30 NUFFT phases, interleaved, full size on one GPU; ~1M sampled
    elements (incl. both ends) vs the oracle on the regenerated inputs."""
    n = inputs.size(4)
    th = gen_to_device(4, n)
    o = torch.empty(2 * n, dtype=torch.float32, device="cuda")
    for variant in VARIANTS:
        sp.sincos_pairs(th, interleaved_out=o, variant=variant)
        torch.cuda.synchronize()
        idx = sampled_indices(n, seed=variant)
        it = torch.from_numpy(idx).cuda()
        ov = o.view(n, 2)[it].cpu().numpy()
        want_th = inputs.generate_at(4, idx.astype(np.uint64))
        assert np.array_equal(th[it].cpu().numpy().view(np.uint32), want_th.view(np.uint32))
        os_, oc = oracle.sincos(want_th, variant)
        assert_parity(ov[:, 1].copy(), ov[:, 0].copy(), os_, oc, "C4")
    del th, o
    torch.cuda.empty_cache()


def test_c5_full_size_sampled_and_sharded():
    """BASELINE configs[4]: 2^32 N(0, 100^2) (16 GiB in, 32 GiB out) on one GPU with 64-bit
    indexing; sampled elements vs the oracle; then the same array as 8 contiguous shards
    (sincos_pairs_sharded, all on this device) must reproduce the one-shot output bit for bit."""
    n = inputs.size(5)
    th = gen_to_device(5, n)
    s = torch.empty(n, dtype=torch.float32, device="cuda")
    c = torch.empty(n, dtype=torch.float32, device="cuda")
    variant = oracle.VARIANT_A
    sp.sincos_pairs(th, s, c, variant=variant)
    torch.cuda.synchronize()
    idx = sampled_indices(n, seed=5)
    it = torch.from_numpy(idx).cuda()
    want_th = inputs.generate_at(5, idx.astype(np.uint64))
    assert np.array_equal(th[it].cpu().numpy().view(np.uint32), want_th.view(np.uint32))
    os_, oc = oracle.sincos(want_th, variant)
    assert_parity(s[it].cpu().numpy(), c[it].cpu().numpy(), os_, oc, "C5")
    # elements past 2^31 and 2^32-1 exist and are not garbage
    assert int(idx.max()) == n - 1
    # sharded run into fresh buffers
    s2 = torch.empty_like(s)
    c2 = torch.empty_like(c)
    G = 8
    shards = []
    for g in range(G):
        lo, hi = sp.shard_range(n, G, g)
        shards.append({"theta": th[lo:hi], "sin": s2[lo:hi], "cos": c2[lo:hi]})
    sp.sincos_pairs_sharded(shards, variant=variant)
    torch.cuda.synchronize()
    assert torch.equal(s.view(torch.int32), s2.view(torch.int32))
    assert torch.equal(c.view(torch.int32), c2.view(torch.int32))
    del th, s, c, s2, c2
    torch.cuda.empty_cache()


# ---- whole input space -------------------------------------------------------------

M1 = 0x9E3779B97F4A7C15
M2 = 0xBF58476D1CE4E5B9
M3 = 0x94D049BB133111EB
MU = 0xD6E8FEB86659FD93


def _s64(x):
    return x - (1 << 64) if x >= (1 << 63) else x


def _lsr(z, k):
    return (z >> k) & ((1 << (64 - k)) - 1)


def _hash_chunk(u0, s, c):
    """The SURVEY [X13] hash of GPU outputs, computed with torch int64 ops on the device
    (test-side code; wrapping 64-bit arithmetic)."""
    n = s.numel()
    sb = s.view(torch.int32).to(torch.int64) & 0xFFFFFFFF
    cb = c.view(torch.int32).to(torch.int64) & 0xFFFFFFFF
    sb = torch.where(torch.isnan(s), torch.full_like(sb, 0x7FC00000), sb)
    cb = torch.where(torch.isnan(c), torch.full_like(cb, 0x7FC00000), cb)
    sb = torch.where(s == 0, torch.zeros_like(sb), sb)
    cb = torch.where(c == 0, torch.zeros_like(cb), cb)
    key = (sb << 32) | cb
    u = torch.arange(u0, u0 + n, dtype=torch.int64, device=s.device)
    z = key ^ (u * _s64(MU))
    z = z + _s64(M1)
    z = (z ^ _lsr(z, 30)) * _s64(M2)
    z = (z ^ _lsr(z, 27)) * _s64(M3)
    z = z ^ _lsr(z, 31)
    h = int(z.sum().item()) % (1 << 64)
    nan = int((torch.isnan(s) | torch.isnan(c)).sum().item())
    ex = int(((s == 0) & (c == 1)).sum().item())
    return h, nan, ex


def test_hash_helper_matches_oracle_hash():
    """The torch hash above equals the oracle's C hash on the same outputs (host copy)."""
    u0 = 0x3F000000
    th = np.arange(u0, u0 + (1 << 16), dtype=np.uint32).view(np.float32)
    s, c = oracle.sincos(th, 0)
    h, _, _ = _hash_chunk(u0, torch.from_numpy(s).cuda(), torch.from_numpy(c).cuda())
    assert h == oracle.hash_outputs(s=s, c=c, first_bits=u0)


@pytest.mark.parametrize("variant,name", [(oracle.VARIANT_N, "N"), (oracle.VARIANT_A, "A")])
def test_all_fp32_bit_patterns(golden, variant, name):
    """Every one of the 2^32 fp32 inputs: the hash, NaN count and exact-(0,1) count of the GPU
    outputs equal the oracle's committed whole-space run (tests/golden/oracle_exhaustive.json),
    which equals the survey's independent transcription [X13]."""
    import json
    run_ = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "oracle_exhaustive.json")))
    want = run_[name]["all_bits"]
    assert want["hash"] == golden["survey_crosscheck"]["all_bits_hash"][name]
    chunk = 1 << 28
    s = torch.empty(chunk, dtype=torch.float32, device="cuda")
    c = torch.empty(chunk, dtype=torch.float32, device="cuda")
    H, NN, EX = 0, 0, 0
    for u0 in range(0, 1 << 32, chunk):
        th = torch.arange(u0, u0 + chunk, dtype=torch.int64, device="cuda").to(torch.int32).view(torch.float32)
        sp.sincos_pairs(th, s, c, variant=variant)
        h, nn, ex = _hash_chunk(u0, s, c)
        H, NN, EX = (H + h) % (1 << 64), NN + nn, EX + ex
    assert "0x%016X" % H == want["hash"]
    assert NN == want["nan_pairs"] and EX == want["exact_0_1"]


def test_reciprocal_exhaustive():
    """Reading G3: the kernel's reciprocal equals IEEE RN(1/d) (CPU 1.0f/d) for every fp32 d in
    [0.5, 2), which contains every s2^2 + c2^2 the method produces ([X10])."""
    d = np.arange(0x3F000000, 0x40000000, dtype=np.uint32).view(np.float32)
    want = np.float32(1.0) / d
    dt = torch.from_numpy(d).cuda()
    out = torch.empty_like(dt)
    sp.debug_reciprocal(dt, out)
    got = out.cpu().numpy()
    bad = np.flatnonzero(got.view(np.uint32) != want.view(np.uint32))
    assert bad.size == 0, (bad.size, d[bad[:5]])


# ---- edge cases: lengths, alignment, in-place, every kernel instance ------------------

def test_lengths_and_alignments():
    """lengths 0..257 at every element offset 0..7 of theta and outputs, shared
    (vector path with scalar head/tail) and unshared (scalar path) alignment, both layouts."""
    rng = np.random.default_rng(11)
    base = rng.uniform(-50, 50, 4096).astype(np.float32)
    ref = {v: oracle.sincos(base, v) for v in VARIANTS}
    big_t = torch.from_numpy(base).cuda()
    big_s = torch.empty(4096 + 64, dtype=torch.float32, device="cuda")
    big_c = torch.empty(4096 + 64, dtype=torch.float32, device="cuda")
    big_i = torch.empty(2 * 4096 + 64, dtype=torch.float32, device="cuda")
    for variant in VARIANTS:
        rs, rc = ref[variant]
        for n in list(range(0, 258)) + [1000, 4000]:
            for (ot, oo) in ((0, 0), (1, 1), (3, 3), (5, 5), (7, 7), (1, 0), (0, 3), (2, 6)):
                if ot + n > 4096:
                    continue
                t = big_t[ot:ot + n]
                s = big_s[oo:oo + n]
                c = big_c[oo + 32:oo + 32 + n] if n <= 4096 - 32 else None
                if c is None:
                    continue
                sp.sincos_pairs(t, s, c, variant=variant)
                io = big_i[2 * oo:2 * oo + 2 * n]
                sp.sincos_pairs(t, interleaved_out=io, variant=variant)
                torch.cuda.synchronize()
                assert_parity(s.cpu().numpy(), c.cpu().numpy(), rs[ot:ot + n], rc[ot:ot + n], f"n={n} off={ot},{oo}")
                iv = io.cpu().numpy()
                assert_parity(iv[1::2], iv[0::2], rs[ot:ot + n], rc[ot:ot + n], f"inter n={n} off={ot},{oo}")


@pytest.mark.parametrize("variant", VARIANTS)
def test_in_place(variant):
    th = inputs.generate(1, 0, (1 << 16) + 5)
    os_, oc = oracle.sincos(th, variant)
    t = torch.from_numpy(th).cuda()
    c = torch.empty_like(t)
    sp.sincos_pairs(t, t, c, variant=variant)           # sin overwrites theta
    torch.cuda.synchronize()
    assert_parity(t.cpu().numpy(), c.cpu().numpy(), os_, oc, "in-place sin")
    t = torch.from_numpy(th).cuda()
    s = torch.empty_like(t)
    sp.sincos_pairs(t, s, t, variant=variant)           # cos overwrites theta
    torch.cuda.synchronize()
    assert_parity(s.cpu().numpy(), t.cpu().numpy(), os_, oc, "in-place cos")


@pytest.mark.parametrize("threads", [128, 256, 512])
@pytest.mark.parametrize("vec", [4, 8])
@pytest.mark.parametrize("unroll", [1, 2, 4])
@pytest.mark.parametrize("prefetch", [0, 1])
def test_every_kernel_instance(threads, vec, unroll, prefetch):
    """Every (threads, vector width, unroll, prefetch) of the A/B build (the product runs the
    first of them, 128 / 8 / 1 / 0, full grid), both variants and layouts, on a ragged size,
    with a 1-block-per-SM grid (many grid-stride trips), the occupancy grid, and the full
    grid (about one trip per thread)."""
    th = inputs.generate(2, 12345, (1 << 20) + 13)
    want = {v: oracle.sincos(th, v) for v in VARIANTS}
    for bps in (0, 1, 6):
        with ab.knobs(launch=(threads, bps, vec, unroll, prefetch)):
            for variant in VARIANTS:
                for inter in (False, True):
                    s, c = run(th, variant, inter)
                    assert_parity(s, c, *want[variant],
                                  f"t{threads} v{vec} u{unroll} pf{prefetch} bps{bps} inter={inter}")


def test_special_values_gpu():
    th = np.array([0.0, -0.0, np.nan, np.inf, -np.inf, 1e-45, -1e-45, 1e-40, 3.4e38, -3.4e38,
                   math.pi, -math.pi, math.pi / 2, 1e30] * 3, dtype=np.float32)
    for variant in VARIANTS:
        s, c = run(th, variant)
        os_, oc = oracle.sincos(th, variant)
        assert_parity(s, c, os_, oc, "special")
        assert np.isnan(s[2]) and np.isnan(c[3]) and np.isnan(s[4])


# ---- host path, stats kernel, null kernel, launch accounting ---------------------------

@pytest.mark.parametrize("inter", [False, True])
@pytest.mark.parametrize("ws_mib", [0, 64])
def test_host_buffer_path(inter, ws_mib):
    """sincos_pairs_host (chunked H2D -> kernel -> D2H over three streams) equals the oracle;
    the minimum workspace forces many 2^16-element chunks and a ragged last one, a 64 MiB one
    the whole ramp of chunk sizes (2^16, 2^17, ... up to the slot size) and a ragged end."""
    n = (1 << 21) + 77
    th = inputs.generate(3, 0, n)
    th_h = torch.from_numpy(th).pin_memory()
    ws = torch.empty(max(sp.host_workspace_min_bytes(), ws_mib << 20), dtype=torch.uint8, device="cuda")
    for variant in VARIANTS:
        if inter:
            o = torch.empty(2 * n, dtype=torch.float32).pin_memory()
            sp.sincos_pairs_host(th_h, interleaved_out=o, variant=variant, workspace=ws)
            s, c = o.numpy()[1::2], o.numpy()[0::2]
        else:
            s_h = torch.empty(n, dtype=torch.float32).pin_memory()
            c_h = torch.empty(n, dtype=torch.float32).pin_memory()
            sp.sincos_pairs_host(th_h, s_h, c_h, variant=variant, workspace=ws)
            s, c = s_h.numpy(), c_h.numpy()
        os_, oc = oracle_threaded(th, variant)
        assert_parity(s, c, os_, oc, "host path")


def test_stats_kernel_matches_oracle_metrics():
    """KB5 (fp64 on the device) vs the oracle's P:135-139 metrics with double libm."""
    th = inputs.generate(1)
    for variant in VARIANTS:
        t = torch.from_numpy(th).cuda()
        s, c = torch.empty_like(t), torch.empty_like(t)
        sp.sincos_pairs(t, s, c, variant=variant)
        st = sp.error_stats(t, s, c)
        ref = oracle.error_stats(th, s.cpu().numpy(), c.cpu().numpy())
        assert st["n"] == ref.count and st["nan_count"] == ref.nan_count
        assert abs(st["max_comb"] - ref.max_comb) <= 1e-12
        assert abs(st["rms"] - ref.rms) / ref.rms < 1e-9
        assert abs(st["max_amp"] - ref.max_amp) <= 1e-12
        st2 = sp.error_stats(t, s, c)
        assert st2["raw"] == st["raw"]                       # deterministic
    t = torch.tensor([0.0, float("nan"), float("inf")], device="cuda")
    s, c = torch.empty_like(t), torch.empty_like(t)
    sp.sincos_pairs(t, s, c)
    st = sp.error_stats(t, s, c)
    assert st["n"] == 1 and st["nan_count"] == 2 and st["max_comb"] == 0.0


def test_null_kernel_copies():
    th = inputs.generate(1, 0, 1000003)
    t = torch.from_numpy(th).cuda()
    s, c = torch.empty_like(t), torch.empty_like(t)
    sp.null_4in8out(t, s, c)
    o = torch.empty(2 * t.numel(), device="cuda")
    sp.null_4in8out(t, interleaved_out=o)
    torch.cuda.synchronize()
    assert torch.equal(s, t) and torch.equal(c, t) and torch.equal(o[0::2], t) and torch.equal(o[1::2], t)


def test_host_buffer_path_pageable():
    """sincos_pairs_host on ordinary (pageable) host memory: correct, if slower (the copies stage
    through the driver's pinned buffers)."""
    n = (1 << 20) + 9
    th = inputs.generate(2, 7, n)
    ws = torch.empty(8 << 20, dtype=torch.uint8, device="cuda")
    for variant in VARIANTS:
        s_h, c_h = torch.empty(n), torch.empty(n)
        sp.sincos_pairs_host(torch.from_numpy(th), s_h, c_h, variant=variant, workspace=ws)
        io = torch.empty(2 * n)
        sp.sincos_pairs_host(torch.from_numpy(th), interleaved_out=io, variant=variant, workspace=ws)
        os_, oc = oracle.sincos(th, variant)
        assert_parity(s_h.numpy(), c_h.numpy(), os_, oc, "pageable split")
        assert_parity(io.numpy()[1::2], io.numpy()[0::2], os_, oc, "pageable inter")


def test_launches_are_counted():
    before = sp.launch_count()
    t = torch.zeros(100, device="cuda")
    sp.sincos(t)
    assert sp.launch_count() == before + 1


def test_rejects_cpu_tensors():
    with pytest.raises(ValueError):
        sp.sincos_pairs(torch.zeros(8), torch.zeros(8), torch.zeros(8))


def test_concurrent_host_threads():
    """Thread-safe and reentrant (header): several host threads call the device path
    on their own streams and the host-buffer path at the same time (ctypes drops the GIL, so
    the calls overlap); every result equals the oracle."""
    from concurrent.futures import ThreadPoolExecutor

    n = (1 << 20) + 13
    cases = [(seed, variant, host) for seed in (1, 2, 3) for variant in VARIANTS for host in (False, True)]
    ths = {seed: inputs.generate(seed, 0, n) for seed in (1, 2, 3)}

    def work(case):
        seed, variant, host = case
        th = ths[seed]
        outs = []
        for _ in range(3):
            if host:
                th_h = torch.from_numpy(th).pin_memory()
                s_h = torch.empty(n, dtype=torch.float32).pin_memory()
                c_h = torch.empty(n, dtype=torch.float32).pin_memory()
                ws = torch.empty(sp.host_workspace_min_bytes(), dtype=torch.uint8, device="cuda")
                sp.sincos_pairs_host(th_h, s_h, c_h, variant=variant, workspace=ws)
                outs.append((s_h.numpy().copy(), c_h.numpy().copy()))
            else:
                st = torch.cuda.Stream()
                with torch.cuda.stream(st):
                    t = torch.from_numpy(th).cuda(non_blocking=False)
                    s, c = torch.empty_like(t), torch.empty_like(t)
                    sp.sincos_pairs(t, s, c, variant=variant, stream=st)
                st.synchronize()
                outs.append((s.cpu().numpy(), c.cpu().numpy()))
        return outs

    with ThreadPoolExecutor(len(cases)) as ex:
        results = list(ex.map(work, cases))
    want = {(seed, v): oracle_threaded(ths[seed], v) for seed in (1, 2, 3) for v in VARIANTS}
    for (seed, variant, host), outs in zip(cases, results):
        os_, oc = want[(seed, variant)]
        for s, c in outs:
            assert_parity(s, c, os_, oc, f"thread seed={seed} variant={variant} host={host}")


# ---- unshared alignment: register re-alignment (KB3b) and one element per thread (KB3) ----

@pytest.mark.parametrize("mode", [1, 2])
@pytest.mark.parametrize("bps", [0, 1])
def test_realign_path(bps, mode):
    """theta at every offset mod 4 floats against outputs at every offset: where the outputs
    can take 128-bit stores the re-aligning kernel runs (k = 1, 2, 3 with head peeling when the
    aligned theta base would precede theta); lengths around the vector/tail boundaries and
    large enough for many warps; bps = 1 forces many warp-uniform grid-stride trips."""
    rng = np.random.default_rng(21)
    N = 200_003
    base = rng.uniform(-3000, 3000, N + 64).astype(np.float32)
    ref = {v: oracle.sincos(base, v) for v in VARIANTS}
    big_t = torch.from_numpy(base).cuda()
    big_s = torch.empty(N + 64, dtype=torch.float32, device="cuda")
    big_c = torch.empty(N + 64, dtype=torch.float32, device="cuda")
    big_i = torch.empty(2 * N + 64, dtype=torch.float32, device="cuda")
    # the product (mode 1, full grid) or the A/B build (128-bit form only, grid-stride grids)
    ctx = ab.knobs(blocks_per_sm=bps, realign=mode) if (mode, bps) != (1, 0) else contextlib.nullcontext()
    with ctx:
        for variant in VARIANTS:
            rs, rc = ref[variant]
            for n in list(range(0, 24)) + [127, 128, 129, 1000, 4097, N]:
                for ot in (0, 1, 2, 3, 5):
                    for oo in (0, 1, 2, 3, 6):
                        if (ot - oo) % 4 == 0 and n > 24:
                            continue          # shared alignment: the vector path, tested above
                        t = big_t[ot:ot + n]
                        s = big_s[oo:oo + n]
                        c = big_c[oo + 8:oo + 8 + n] if oo + 8 + n <= N + 64 else big_c[oo:oo + n]
                        sp.sincos_pairs(t, s, c, variant=variant)
                        io = big_i[2 * oo:2 * oo + 2 * n]
                        sp.sincos_pairs(t, interleaved_out=io, variant=variant)
                        torch.cuda.synchronize()
                        assert_parity(s.cpu().numpy(), c.cpu().numpy(), rs[ot:ot + n], rc[ot:ot + n],
                                      f"realign n={n} off={ot},{oo} bps={bps}")
                        iv = io.cpu().numpy()
                        assert_parity(iv[1::2], iv[0::2], rs[ot:ot + n], rc[ot:ot + n],
                                      f"realign inter n={n} off={ot},{oo} bps={bps}")


def test_scalar_path_unshared_outputs():
    """The one-element-per-thread kernel: sin and cos at different offsets mod 16 B, and an
    interleaved output only 4-B aligned (odd float offset); with re-alignment off, every
    unshared case goes there too."""
    rng = np.random.default_rng(22)
    n = 70_001
    base = rng.uniform(-100, 100, n + 16).astype(np.float32)
    big_t = torch.from_numpy(base).cuda()
    big_s = torch.empty(n + 16, dtype=torch.float32, device="cuda")
    big_c = torch.empty(n + 16, dtype=torch.float32, device="cuda")
    big_i = torch.empty(2 * n + 16, dtype=torch.float32, device="cuda")
    for variant in VARIANTS:
        rs, rc = oracle.sincos(base, variant)
        for realign in (True, False):
            with (contextlib.nullcontext() if realign else ab.knobs(realign=0)):
                for ot, os_, oc_, oi in ((0, 1, 2, 1), (1, 0, 3, 3), (2, 2, 2, 2), (3, 0, 0, 5)):
                    t = big_t[ot:ot + n]
                    s, c = big_s[os_:os_ + n], big_c[oc_:oc_ + n]
                    io = big_i[oi:oi + 2 * n]
                    sp.sincos_pairs(t, s, c, variant=variant)
                    sp.sincos_pairs(t, interleaved_out=io, variant=variant)
                    torch.cuda.synchronize()
                    assert_parity(s.cpu().numpy(), c.cpu().numpy(), rs[ot:ot + n], rc[ot:ot + n],
                                  f"scalar off={ot},{os_},{oc_} realign={realign}")
                    iv = io.cpu().numpy()
                    assert_parity(iv[1::2], iv[0::2], rs[ot:ot + n], rc[ot:ot + n],
                                  f"scalar inter off={ot},{oi} realign={realign}")


@pytest.mark.parametrize("variant,name", [(oracle.VARIANT_N, "N"), (oracle.VARIANT_A, "A")])
@pytest.mark.parametrize("path", ["interleaved", "realign_split", "realign_interleaved", "scalar_split",
                                  "outshift_split", "outshift_interleaved", "hybrid_split"])
def test_all_fp32_bit_patterns_other_paths(golden, variant, name, path):
    """The whole-input-space hash through the other kernels: the 256-bit interleaved kernel,
    the re-aligning kernel (theta one float off the outputs; split and interleaved) and the
    one-element-per-thread kernel -- each equals the oracle's committed whole-space run."""
    import json
    run_ = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "oracle_exhaustive.json")))
    want = run_[name]["all_bits"]
    chunk = 1 << 28
    toff = 1 if path in ("realign_split", "realign_interleaved", "scalar_split") else 0
    tbuf = torch.empty(chunk + 8, dtype=torch.float32, device="cuda")
    with (ab.knobs(realign=0) if path == "scalar_split" else contextlib.nullcontext()):
        if "inter" in path:
            ibuf = torch.empty(2 * chunk + 8, dtype=torch.float32, device="cuda")
            io = ibuf[1:1 + 2 * chunk] if path == "outshift_interleaved" else ibuf[:2 * chunk]   # 4-B pairs
        elif path in ("outshift_split", "hybrid_split"):
            sbuf = torch.empty(chunk + 8, dtype=torch.float32, device="cuda")
            cbuf = torch.empty(chunk + 8, dtype=torch.float32, device="cuda")
            if path == "outshift_split":
                s, c = sbuf[1:1 + chunk], cbuf[2:2 + chunk]      # sin and cos apart mod 16 B
            else:
                s, c = sbuf[5:5 + chunk], cbuf[3:3 + chunk]      # both off theta's frame: the hybrid form
        else:
            s = torch.empty(chunk, dtype=torch.float32, device="cuda")
            c = torch.empty(chunk, dtype=torch.float32, device="cuda")
        H, NN, EX = 0, 0, 0
        for u0 in range(0, 1 << 32, chunk):
            th = tbuf[toff:toff + chunk]
            th.view(torch.int32).copy_(torch.arange(u0, u0 + chunk, dtype=torch.int64, device="cuda").to(torch.int32))
            if "inter" in path:
                sp.sincos_pairs(th, interleaved_out=io, variant=variant)
                s, c = io[1::2], io[0::2]
            else:
                sp.sincos_pairs(th, s, c, variant=variant)
            h, nn, ex = _hash_chunk(u0, s.contiguous(), c.contiguous())
            H, NN, EX = (H + h) % (1 << 64), NN + nn, EX + ex
    assert "0x%016X" % H == want["hash"], path
    assert NN == want["nan_pairs"] and EX == want["exact_0_1"]


@pytest.mark.parametrize("variant,name", [(oracle.VARIANT_N, "N"), (oracle.VARIANT_A, "A")])
@pytest.mark.parametrize("path", ["phase_vec", "phase_flat", "method_paper_table"])
def test_all_fp32_bit_patterns_next_kernels(golden, variant, name, path):
    """Every fp32 input through the NEXT-row kernels that evaluate the same pairs: the phase
    grid with f = [1] (p = RN(1 * t) = t exactly, radians; 256-bit row kernel, and the flat
    kernel with t one float off) and the general-method kernel with the paper's own table --
    hash, NaN and exact-(0, 1) counts equal the oracle's whole-space run."""
    import json
    run_ = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "oracle_exhaustive.json")))
    want = run_[name]["all_bits"]
    chunk = 1 << 28
    toff = 1 if path == "phase_flat" else 0
    tbuf = torch.empty(chunk + 8, dtype=torch.float32, device="cuda")
    s = torch.empty(chunk, dtype=torch.float32, device="cuda")
    c = torch.empty(chunk, dtype=torch.float32, device="cuda")
    one = torch.ones(1, dtype=torch.float32, device="cuda")
    m = sp.make_method(*sp.PAPER_METHODS[variant])
    H, NN, EX = 0, 0, 0
    for u0 in range(0, 1 << 32, chunk):
        th = tbuf[toff:toff + chunk]
        th.view(torch.int32).copy_(torch.arange(u0, u0 + chunk, dtype=torch.int64, device="cuda").to(torch.int32))
        if path.startswith("phase"):
            sp.phase_grid(one, th, s, c, units=sp.RADIANS, variant=variant)
        else:
            sp.sincos_pairs_method(th, m, s, c)
        h, nn, ex = _hash_chunk(u0, s, c)
        H, NN, EX = (H + h) % (1 << 64), NN + nn, EX + ex
    assert "0x%016X" % H == want["hash"], path
    assert NN == want["nan_pairs"] and EX == want["exact_0_1"]


def test_cis_complex_view():
    """cis(theta) = e^{i theta} as complex64: real part the method's cos, imaginary its sin."""
    th = inputs.generate(1, 0, 3000).reshape(3, 1000)
    t = torch.from_numpy(th).cuda()
    z = sp.cis(t)
    assert z.dtype == torch.complex64 and z.shape == t.shape
    ws, wc = oracle.sincos(th.ravel(), 0)
    zz = z.cpu().numpy().ravel()
    assert_parity(zz.imag.copy(), zz.real.copy(), ws, wc, "cis")


@pytest.mark.parametrize("which", [3, 4])
@pytest.mark.parametrize("inter", [False, True])
def test_compare_cuda_context_kernels(which, inter):
    """The bench's context kernels (CUDA sincosf / __sincosf in the hot path's kernel shape) run
    and compute sin/cos (loose check against torch's fp64), ragged tail included; misaligned
    buffers are refused."""
    n = (1 << 16) + 5
    t = torch.rand(n, device="cuda", dtype=torch.float32) * 20 - 10
    if inter:
        o = torch.empty(2 * n, device="cuda")
        sp.compare_cuda(t, interleaved_out=o, which=which)
        s, c = o[1::2], o[0::2]
    else:
        s, c = torch.empty_like(t), torch.empty_like(t)
        sp.compare_cuda(t, s, c, which=which)
    torch.cuda.synchronize()
    td = t.double()
    tol = 1e-6 if which == 3 else 1e-5
    assert torch.max(torch.abs(s.double() - torch.sin(td))) < tol
    assert torch.max(torch.abs(c.double() - torch.cos(td))) < tol
    with pytest.raises(sp.SincosError):
        sp.compare_cuda(t[1:], s[1:], c[1:], which=which) if not inter else \
            sp.compare_cuda(t[1:], interleaved_out=o[2:], which=which)


@pytest.mark.parametrize("inter", [False, True])
def test_c5_full_size_realigned(inter):
    """2^32 angles with theta one float off the outputs: the re-aligning kernel over 64-bit
    element indices (every warp's shuffles and the last lanes' own loads past 2^31 and up to
    2^32 - 1); sampled elements vs the oracle, the last element included."""
    n = inputs.size(5)
    tb = torch.empty(n + 8, dtype=torch.float32, device="cuda")
    chunk = 1 << 28
    for off in range(0, n, chunk):
        m = min(chunk, n - off)
        tb[1 + off:1 + off + m].copy_(torch.from_numpy(inputs.generate(5, off, m)))
    th = tb[1:1 + n]
    if inter:
        io = torch.empty(2 * n, dtype=torch.float32, device="cuda")
        sp.sincos_pairs(th, interleaved_out=io, variant=1)
    else:
        s = torch.empty(n, dtype=torch.float32, device="cuda")
        c = torch.empty(n, dtype=torch.float32, device="cuda")
        sp.sincos_pairs(th, s, c, variant=1)
    torch.cuda.synchronize()
    idx = sampled_indices(n, seed=55)
    it = torch.from_numpy(idx).cuda()
    want_th = inputs.generate_at(5, idx.astype(np.uint64))
    os_, oc = oracle.sincos(want_th, 1)
    if inter:
        gs, gc = io[2 * it + 1].cpu().numpy(), io[2 * it].cpu().numpy()
    else:
        gs, gc = s[it].cpu().numpy(), c[it].cpu().numpy()
    assert_parity(gs, gc, os_, oc, f"C5 realigned inter={inter}")
    assert int(idx.max()) == n - 1
    del tb, th
    torch.cuda.empty_cache()


def test_binding_refuses_mixed_devices_and_follows_tensor_device():
    """The binding runs each call on its tensors' device (made current for the call) and refuses
    tensors on two devices; on a 1-GPU box the mixed case is CPU + CUDA (refused as before) and
    the current device is left unchanged."""
    t = torch.rand(100, device="cuda")
    s, c = torch.empty_like(t), torch.empty_like(t)
    cur = torch.cuda.current_device()
    sp.sincos_pairs(t, s, c)
    assert torch.cuda.current_device() == cur
    with pytest.raises(ValueError):
        sp.sincos_pairs(t, torch.empty(100), c)
    if torch.cuda.device_count() > 1:
        t1 = torch.rand(100, device="cuda:1")
        with pytest.raises(ValueError):
            sp.sincos_pairs(t1, s, c)
        s1, c1 = torch.empty_like(t1), torch.empty_like(t1)
        sp.sincos_pairs(t1, s1, c1)                    # runs on device 1 though 0 is current
        torch.cuda.synchronize(1)
        ws, wc = oracle.sincos(t1.cpu().numpy(), 0)
        assert_parity(s1.cpu().numpy(), c1.cpu().numpy(), ws, wc, "device 1")


@pytest.mark.parametrize("pdl", [True, False])
def test_dependent_launch_chain_keeps_stream_order(pdl):
    """Programmatic dependent launch must not let a kernel read its predecessor's output early:
    a chain of 12 back-to-back launches, each reading the previous one's sin output (in place
    every other step), no host sync in between, equals the oracle applied 12 times."""
    with (contextlib.nullcontext() if pdl else ab.knobs(pdl=0)):
        n = (1 << 22) + 3
        th = inputs.generate(1, 0, n)
        cur = torch.from_numpy(th).cuda()
        c = torch.empty_like(cur)
        want = th
        for k in range(12):
            v = k % 2
            if k % 2 == 0:
                nxt = torch.empty_like(cur)
                sp.sincos_pairs(cur, nxt, c, variant=v)
                cur = nxt
            else:
                sp.sincos_pairs(cur, cur, c, variant=v)         # in place: sin over theta
            want, wc = oracle.sincos(want, v)
        torch.cuda.synchronize()
        assert_parity(cur.cpu().numpy(), c.cpu().numpy(), want, wc, f"chain pdl={pdl}")


@pytest.mark.parametrize("bps", [1, 2])
def test_in_place_realigning_many_trips(bps):
    """The in-place read-only-load invariant under grid-stride: on the A/B build with 1-2 blocks
    per SM every thread makes hundreds of trips, so a thread that read an element some other
    thread had already overwritten (or a stale cached line) would show up as a mismatch against
    the out-of-place run.  theta == sin and theta == cos, the other output at every offset."""
    th = inputs.generate(2, 3, (1 << 22) + 5)
    want = {v: oracle.sincos(th, v) for v in VARIANTS}
    with ab.knobs(blocks_per_sm=bps):
        for variant in VARIANTS:
            os_, oc = want[variant]
            for off in (1, 2, 3, 4, 5, 6, 7):
                t = torch.from_numpy(th).cuda()
                ob = torch.empty(t.numel() + 8, device="cuda")
                o = ob[off:off + t.numel()]
                sp.sincos_pairs(t, t, o, variant=variant)              # sin over theta
                torch.cuda.synchronize()
                assert_parity(t.cpu().numpy(), o.cpu().numpy(), os_, oc, f"sin in place, cos +{off}, bps={bps}")
                t = torch.from_numpy(th).cuda()
                sp.sincos_pairs(t, o, t, variant=variant)              # cos over theta
                torch.cuda.synchronize()
                assert_parity(o.cpu().numpy(), t.cpu().numpy(), os_, oc, f"cos in place, sin +{off}, bps={bps}")


@pytest.mark.parametrize("variant", VARIANTS)
@pytest.mark.parametrize("soff", [1, 2, 3, 6])
def test_in_place_cos_over_theta_with_sin_off_alignment(variant, soff):
    """theta == cos_out with sin at another offset (the mirror of the case below): through the
    output-realigning kernel, at a size of many warps and a ragged tail."""
    th = inputs.generate(5, 0, (1 << 21) + 13)
    os_, oc = oracle.sincos(th, variant)
    t = torch.from_numpy(th).cuda()
    sb = torch.empty(t.numel() + 8, device="cuda")
    s = sb[soff:soff + t.numel()]
    sp.sincos_pairs(t, s, t, variant=variant)
    torch.cuda.synchronize()
    assert_parity(s.cpu().numpy(), t.cpu().numpy(), os_, oc, f"in place cos, sin +{soff}")


@pytest.mark.parametrize("variant", VARIANTS)
@pytest.mark.parametrize("coff", [1, 2, 3, 5])
def test_in_place_with_cos_off_alignment(variant, coff):
    """theta == sin_out (exact in place) with cos at another offset: the output-realigning
    kernel reads theta through the read-only path while writing sin over it, one owner thread
    per element -- still the oracle's pairs."""
    th = inputs.generate(2, 0, (1 << 20) + 11)
    os_, oc = oracle.sincos(th, variant)
    t = torch.from_numpy(th).cuda()
    cb = torch.empty(t.numel() + 8, device="cuda")
    c = cb[coff:coff + t.numel()]
    sp.sincos_pairs(t, t, c, variant=variant)
    torch.cuda.synchronize()
    assert_parity(t.cpu().numpy(), c.cpu().numpy(), os_, oc, f"in place, cos +{coff}")


@pytest.mark.parametrize("variant", VARIANTS)
def test_outshift_interleaved_two_trips(variant):
    """KB3c for interleaved pairs at k = 3, 5, 7 floats runs two trips per thread with the next
    trip's theta vector prefetched (half the blocks; csrc/sincos_outshift.cu outshift_pf):
    every odd interleaved offset against an aligned and an unaligned theta, at sizes where the
    last block has one trip, a partial second trip, exactly two, and a ragged tail -- and on
    the A/B build's grid-stride grids (hundreds of trips per thread)."""
    rng = np.random.default_rng(77)
    N = 1 << 20
    base = rng.uniform(-5e3, 5e3, N + 64).astype(np.float32)
    rs, rc = oracle.sincos(base, variant)
    bt = torch.from_numpy(base).cuda()
    bi = torch.empty(2 * N + 64, dtype=torch.float32, device="cuda")
    sizes = [1023, 1024 + 7, 2048, 2048 + 8 * 128 + 3, 8 * 128 * 3 + 1, 8 * 128 * 2 * 77 + 8 * 5 + 6, N]
    for ctx in (contextlib.nullcontext(), ab.knobs(blocks_per_sm=1), ab.knobs(blocks_per_sm=3)):
        with ctx:
            for ot in (0, 8, 3):
                for oi in (1, 3, 5, 7):
                    for n in sizes:
                        t = bt[ot:ot + n]
                        io = bi[oi:oi + 2 * n]
                        io.fill_(float("nan"))
                        sp.sincos_pairs(t, interleaved_out=io, variant=variant)
                        torch.cuda.synchronize()
                        iv = io.cpu().numpy()
                        assert_parity(iv[1::2], iv[0::2], rs[ot:ot + n], rc[ot:ot + n],
                                      f"inter +{oi} theta +{ot} n={n}")
