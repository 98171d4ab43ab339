"""Performance floors (``pytest -m gpu``): each kernel path at ~88% of what DESIGN.md records on
one B200, so a regression of >= 12% in any path fails a test rather than going unnoticed (the
programmatic-dependent-launch change once cost the 128-bit path 15%; only a probe caught it).
HBM-bound paths do not depend on the SM clock, so power capping does not trip them."""
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_cs_0406049_b200 as sp  # noqa: E402

N = 1 << 27


@pytest.fixture(scope="module", autouse=True)
def cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    yield


def gbps(fn, nbytes, reps=10):
    for _ in range(3):
        fn()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return nbytes / (a.elapsed_time(b) / reps / 1e3) / 1e9


@pytest.fixture(scope="module")
def bufs():
    base = torch.rand(N + 16, device="cuda") * 2e4 - 1e4
    sb, cb = torch.empty(N + 16, device="cuda"), torch.empty(N + 16, device="cuda")
    ib = torch.empty(2 * N + 16, device="cuda")
    yield base, sb, cb, ib
    del base, sb, cb, ib
    torch.cuda.empty_cache()


# (theta offset, sin offset, cos offset, interleaved float offset or None, floor GB/s, recorded GB/s)
CASES = {
    "aligned split (256-bit)": (0, 0, 0, None, 6000, 6870),
    "aligned interleaved": (0, 0, 0, 0, 6000, 6890),
    "shared 16 B (256-bit theta re-alignment)": (4, 0, 0, None, 6000, 6800),
    "theta realigned (KB3b)": (1, 0, 0, None, 6000, 6810),
    "theta realigned interleaved": (1, 0, 0, 0, 6000, 6890),
    "outputs realigned (KB3c)": (0, 1, 2, None, 5900, 6760),
    "outputs realigned, sin 4 off (KB3c, cos stored first)": (0, 4, 2, None, 5900, 6600),
    "sin/cos sharing 16 B (hybrid KB3c)": (0, 3, 7, None, 5800, 6570),
    "both streams off theta (hybrid KB3c)": (0, 6, 5, None, 5800, 6570),
    "pairs 4-B only, k = 1 (KB3c)": (0, 0, 0, 1, 5900, 6710),
    "pairs 4-B only, k = 3 (KB3c, two trips)": (0, 0, 0, 3, 5900, 6690),
    "pairs 4-B only, k = 5 (KB3c, two trips)": (0, 0, 0, 5, 5800, 6540),
    "pairs 4-B only, k = 7 (KB3c, two trips)": (0, 0, 0, 7, 5900, 6730),
}


@pytest.mark.parametrize("name", list(CASES))
def test_hot_path_floor(bufs, name):
    """Variant N at C2 size; `recorded` is the r02 sweep's (tools/ab_layouts.py), ~2% run to run."""
    base, sb, cb, ib = bufs
    ot, os_, oc, inter, floor, _ = CASES[name]
    th = base[ot:ot + N]
    if inter is not None:
        o = ib[inter:inter + 2 * N]
        fn = lambda: sp.sincos_pairs(th, interleaved_out=o)  # noqa: E731
    else:
        s, c = sb[os_:os_ + N], cb[oc:oc + N]
        fn = lambda: sp.sincos_pairs(th, s, c)  # noqa: E731
    got = gbps(fn, 12 * N)
    assert got >= floor, f"{name}: {got:.0f} GB/s < floor {floor}"


def test_phase_grid_floor():
    f = torch.rand(1 << 13, device="cuda") * 512
    t = torch.rand(1 << 14, device="cuda")
    o = torch.empty(2 * (1 << 27), device="cuda")
    got = gbps(lambda: sp.phase_grid(f, t, interleaved_out=o, units=sp.TURNS), 8 * (1 << 27))
    assert got >= 6500, got                        # recorded 7.5-7.6 TB/s (write-only ceiling)


def test_phase_grid_short_and_tiny_rows_floor():
    """Ragged short rows (nt = 1001, interleaved: recorded 6.9-7.1 TB/s in the bench) and rows of
    one pair (the tiny-row kernel: recorded 4.6 TB/s written = 6.9 TB/s with the f reads)."""
    f = torch.rand((1 << 27) // 1001, device="cuda") * 512
    t = torch.rand(1001, device="cuda")
    n = f.numel() * 1001
    o = torch.empty(2 * n, device="cuda")
    got = gbps(lambda: sp.phase_grid(f, t, interleaved_out=o, units=sp.TURNS), 8 * n)
    assert got >= 5500, f"nt=1001 {got:.0f}"   # (6.0-6.4 once the board is in its power cap)
    f5 = torch.rand((1 << 27) // 5, device="cuda") * 512       # rows of 5 pairs: the staged kernel
    t5 = torch.rand(5, device="cuda")
    n5 = f5.numel() * 5
    o5 = torch.empty(2 * n5, device="cuda")
    got = gbps(lambda: sp.phase_grid(f5, t5, interleaved_out=o5, units=sp.TURNS), 8 * n5)
    assert got >= 5300, f"nt=5 {got:.0f} (recorded 6.1 TB/s written)"
    f12 = torch.rand((1 << 27) // 12, device="cuda") * 512     # interleaved rows of 12: staged, 2 rows per lane
    t12 = torch.rand(12, device="cuda")
    n12 = f12.numel() * 12
    o12 = torch.empty(2 * n12, device="cuda")
    got = gbps(lambda: sp.phase_grid(f12, t12, interleaved_out=o12, units=sp.TURNS), 8 * n12)
    assert got >= 5600, f"nt=12 {got:.0f} (recorded 6.5 TB/s written)"
    f1 = torch.rand(1 << 27, device="cuda")
    t1 = torch.rand(1, device="cuda")
    s, c = torch.empty(1 << 27, device="cuda"), torch.empty(1 << 27, device="cuda")
    got = gbps(lambda: sp.phase_grid(f1, t1, s, c, units=sp.TURNS), 12 * (1 << 27))
    assert got >= 6000, f"nt=1 {got:.0f} (12 B/pair incl. the f read)"


def test_layout_adapters_floor():
    """sincos_interleave / sincos_deinterleave, 32-B aligned (recorded 6.95-6.98 TB/s, 16 B/elem)."""
    n = 1 << 27
    s, c = torch.rand(n, device="cuda"), torch.rand(n, device="cuda")
    io = torch.empty(2 * n, device="cuda")
    got = gbps(lambda: sp.interleave(s, c, io), 16 * n)
    assert got >= 6000, f"interleave {got:.0f}"
    got = gbps(lambda: sp.deinterleave(io, s, c), 16 * n)
    assert got >= 6000, f"deinterleave {got:.0f}"


def test_fused_sum_floor():
    nf = nt = 1 << 15                              # the C4 shape the number is recorded on
    f = torch.rand(nf, device="cuda") * 512
    t = torch.rand(nt, device="cuda")
    a = torch.randn(nt, dtype=torch.complex64, device="cuda")
    out = torch.empty(nf, dtype=torch.complex64, device="cuda")
    ws = torch.empty(sp.lib().sincos_nudft_workspace_bytes(nf, nt), dtype=torch.uint8, device="cuda")
    terms_per_s = gbps(lambda: sp.nudft(f, t, a, out=out, units=sp.TURNS, workspace=ws), nf * nt) * 1e9
    assert terms_per_s >= 1.0e12, terms_per_s      # recorded 1.31 T terms/s (ALU-bound: margin for the SM clock)


def test_16bit_and_method_floors(bufs):
    base, sb, cb, ib = bufs
    th = base[:N]
    s16 = torch.empty(N, dtype=torch.float16, device="cuda")
    c16 = torch.empty(N, dtype=torch.float16, device="cuda")
    got = gbps(lambda: sp.sincos_pairs_dtype(th, s16, c16), 8 * N)
    assert got >= 6000, f"fp16 {got:.0f}"           # recorded 6.83-6.86 TB/s
    m = sp.make_method(*sp.PAPER_METHODS[0])
    got = gbps(lambda: sp.sincos_pairs_method(th, m, sb[:N], cb[:N]), 12 * N)
    assert got >= 6000, f"method {got:.0f}"         # recorded 6.83-6.89 TB/s
    tb = base[1:1 + N]                                # theta one float off: the re-aligning instances
    got = gbps(lambda: sp.sincos_pairs_dtype(tb, s16, c16), 8 * N)
    assert got >= 5600, f"fp16 realigned {got:.0f}"  # recorded 6.47 TB/s
    got = gbps(lambda: sp.sincos_pairs_method(tb, m, sb[:N], cb[:N]), 12 * N)
    assert got >= 6000, f"method realigned {got:.0f}"  # recorded 6.82 TB/s
    c16b = torch.empty(N + 8, dtype=torch.float16, device="cuda")
    for oc in (1, 2, 4):                              # cos[] off sin[]'s 16-B frame: shuffles / 8-B pieces
        got = gbps(lambda: sp.sincos_pairs_dtype(th, s16, c16b[oc:oc + N]), 8 * N)
        assert got >= 5300, f"fp16 cos+{oc} {got:.0f}"  # recorded 6.0-6.1 (1, 2) / 6.87 (4) TB/s


def test_batched_floor():
    """1000 arrays of 4096 angles in one batched call of the A/B build (recorded 24 us = 169 G
    pairs/s)."""
    from paper_cs_0406049_b200 import ab
    count, n = 1000, 4096
    base = torch.rand(count * n, device="cuda")
    s, c = torch.empty_like(base), torch.empty_like(base)
    ts = [base[i * n:(i + 1) * n] for i in range(count)]
    ss = [s[i * n:(i + 1) * n] for i in range(count)]
    cs = [c[i * n:(i + 1) * n] for i in range(count)]
    table = ab.BatchTable(ts, ss, cs)                 # per-item marshalling paid once
    pairs_per_s = gbps(table.run, count * n, reps=200) * 1e9   # host-bound: ~26 us per call
    assert pairs_per_s >= 8e10, pairs_per_s


def test_phase_grid_ragged_floor():
    """Rows that are not whole vectors (the flat kernel): recorded 6.3-6.5 TB/s at nt = 2^15 - 1."""
    f = torch.rand(1 << 13, device="cuda") * 512
    t = torch.rand((1 << 15) - 1, device="cuda")
    n = (1 << 13) * ((1 << 15) - 1)
    o = torch.empty(2 * n, device="cuda")
    got = gbps(lambda: sp.phase_grid(f, t, interleaved_out=o, units=sp.TURNS), 8 * n)
    assert got >= 5500, got
