"""The Python binding's argument checks (it only marshals, but the library trusts the sizes it
is given): every output's element count, dtype, device side and contiguity are checked before
the C call, so a short or misplaced buffer raises instead of being written past its end; and
temporaries used on a caller-given stream stay valid.  ``pytest -m gpu``."""
import numpy as np
import pytest

import inputs
import oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_cs_0406049_b200 as sp  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    yield


def dev(n, dtype=torch.float32):
    return torch.empty(n, dtype=dtype, device="cuda")


def test_short_outputs_raise_before_any_launch():
    n = 1000
    t = torch.rand(n, device="cuda")
    before = sp.launch_count()
    with pytest.raises(ValueError, match="must hold"):
        sp.sincos_pairs(t, dev(n - 1), dev(n))
    with pytest.raises(ValueError, match="must hold"):
        sp.sincos_pairs(t, interleaved_out=dev(2 * n - 2))
    m = sp.make_method(*sp.PAPER_METHODS[0])
    with pytest.raises(ValueError, match="must hold"):
        sp.sincos_pairs_method(t, m, dev(n), dev(n - 8))
    with pytest.raises(ValueError, match="must hold"):
        sp.sincos_pairs_method(t, m, interleaved_out=dev(n))
    with pytest.raises(ValueError, match="must hold"):
        sp.sincos_pairs_dtype(t, dev(n, torch.float16), dev(n - 1, torch.float16))
    with pytest.raises(TypeError):
        sp.sincos_pairs_dtype(t, dev(n, torch.float16), dev(n, torch.bfloat16))
    with pytest.raises(ValueError, match="must hold"):
        sp.interleave(dev(n), dev(n), dev(2 * n - 1))
    with pytest.raises(ValueError, match="must hold"):
        sp.interleave(dev(n), dev(n - 1), dev(2 * n))
    with pytest.raises(ValueError, match="must hold"):
        sp.deinterleave(dev(2 * n - 2), dev(n), dev(n))
    with pytest.raises(ValueError, match="must hold"):
        sp.phase_grid(dev(3), dev(5), dev(15), dev(14))
    f, tt = torch.rand(8, device="cuda"), torch.rand(16, device="cuda")
    a = torch.zeros(16, dtype=torch.complex64, device="cuda")
    with pytest.raises(ValueError, match="must hold"):
        sp.nudft(f, tt, a, out=torch.empty(7, dtype=torch.complex64, device="cuda"))
    with pytest.raises(ValueError, match="must hold"):
        sp.nudft(f, tt, a[:15])
    with pytest.raises(ValueError, match="must hold"):
        sp.error_stats(t, dev(n), dev(n + 1))
    with pytest.raises(ValueError, match="must hold"):
        sp.sincos_pairs_sharded([{"theta": t, "sin": dev(n), "cos": dev(n - 1)}])
    with pytest.raises(ValueError, match="must hold"):
        sp.null_4in8out(t, interleaved_out=dev(n))
    torch.cuda.synchronize()
    assert sp.launch_count() == before


def test_host_path_requires_host_buffers():
    n = 4096
    th = torch.rand(n).pin_memory()
    ws = torch.empty(sp.host_workspace_min_bytes(), dtype=torch.uint8, device="cuda")
    with pytest.raises(ValueError, match="host"):
        sp.sincos_pairs_host(th, dev(n), torch.empty(n), workspace=ws)      # a device 'host' buffer
    with pytest.raises(ValueError, match="host"):
        sp.sincos_pairs_host(th.cuda(), torch.empty(n), torch.empty(n), workspace=ws)
    with pytest.raises(ValueError, match="must hold"):
        sp.sincos_pairs_host(th, torch.empty(n), torch.empty(n - 1), workspace=ws)
    with pytest.raises(ValueError, match="must hold"):
        sp.sincos_pairs_host(th, interleaved_out=torch.empty(n), workspace=ws)
    with pytest.raises(ValueError, match="workspace"):
        sp.sincos_pairs_host(th, torch.empty(n), torch.empty(n), workspace=torch.empty(1 << 20))


def test_non_contiguous_out_is_refused():
    t = torch.rand(1000, device="cuda")
    s, c = dev(2000)[::2], dev(2000)[::2]
    with pytest.raises(ValueError, match="contiguous"):
        sp.sincos(t, out=(s, c))
    o = torch.empty(1000, 4, device="cuda")[:, :2]
    with pytest.raises(ValueError, match="contiguous"):
        sp.sincos(t, interleaved=True, out=o)
    with pytest.raises(ValueError, match="contiguous"):
        sp.sincos_turns(t, out=(s, c))
    # a strided INPUT is fine (read through a contiguous copy), also a transposed one
    tt = torch.rand(64, 32, device="cuda").t()
    s4, c4 = sp.sincos(tt)
    ws4, wc4 = oracle.sincos(tt.contiguous().cpu().numpy().ravel(), 0)
    assert s4.is_contiguous() and np.array_equal(s4.cpu().numpy().ravel(), ws4)
    assert np.array_equal(c4.cpu().numpy().ravel(), wc4)
    tin = torch.rand(100, 2, device="cuda")[:, 0]
    s3, c3 = sp.sincos(tin)
    ws3, wc3 = oracle.sincos(tin.contiguous().cpu().numpy(), 0)
    assert np.array_equal(s3.cpu().numpy(), ws3) and np.array_equal(c3.cpu().numpy(), wc3)
    # contiguous outs of any shape are filled in place
    s2, c2 = torch.empty(10, 100, device="cuda"), torch.empty(10, 100, device="cuda")
    r = sp.sincos(t.view(10, 100), out=(s2, c2))
    ws, wc = oracle.sincos(t.cpu().numpy(), 0)
    assert r[0] is s2 and np.array_equal(s2.cpu().numpy().ravel(), ws) and np.array_equal(c2.cpu().numpy().ravel(), wc)


def test_temporaries_on_a_side_stream():
    """Calls on a caller-given stream whose temporaries (workspace, contiguous copy of a,
    turns' one-element f, outputs) the binding allocates on the current stream: the results
    equal the current-stream ones even while the current stream keeps allocating."""
    side = torch.cuda.Stream()
    rng = np.random.default_rng(3)
    f = torch.from_numpy(rng.uniform(0, 512, 300).astype(np.float32)).cuda()
    t = torch.from_numpy(rng.uniform(0, 1, 5000).astype(np.float32)).cuda()
    a = torch.from_numpy((rng.normal(size=5000) + 1j * rng.normal(size=5000)).astype(np.complex64)).cuda()
    want = sp.nudft(f, t, a, units=sp.TURNS)
    x = torch.from_numpy(inputs.generate(1, 0, 1 << 20)).cuda()
    ws_, wc_ = sp.sincos_turns(x)
    torch.cuda.synchronize()
    side.wait_stream(torch.cuda.current_stream())
    for _ in range(3):
        got = sp.nudft(f, t, a, units=sp.TURNS, stream=side)
        s, c = sp.sincos_turns(x, stream=side)
        junk = [torch.rand(1 << 20, device="cuda") for _ in range(8)]   # current-stream churn
        del junk
        side.synchronize()
        assert torch.equal(got, want) and torch.equal(s, ws_) and torch.equal(c, wc_)


def test_every_entry_point_accepts_empty_inputs():
    """n = 0 (and nf or nt = 0) is a no-op everywhere: nothing launched, nothing raised; an empty
    sum zeroes its output."""
    e = torch.empty(0, device="cuda")
    before = sp.launch_count()
    sp.sincos_pairs(e, e, e)
    sp.sincos_pairs(e, interleaved_out=e)
    s, c = sp.sincos(e)
    assert s.numel() == 0 and c.numel() == 0
    assert sp.cis(e).numel() == 0
    sp.sincos_pairs_method(e, sp.make_method(*sp.PAPER_METHODS[1]), e, e)
    sp.sincos_pairs_dtype(e, torch.empty(0, dtype=torch.float16, device="cuda"),
                          torch.empty(0, dtype=torch.float16, device="cuda"))
    sp.interleave(e, e, e)
    sp.deinterleave(e, e, e)
    sp.phase_grid(e, torch.rand(5, device="cuda"), e, e)
    sp.phase_grid(torch.rand(5, device="cuda"), e, interleaved_out=e)
    s2, c2 = sp.sincos_turns(e)
    assert s2.numel() == 0
    sp.sincos_pairs_sharded([{"theta": e, "sin": e, "cos": e}])
    sp.sincos_pairs_host(torch.empty(0), torch.empty(0), torch.empty(0),
                         workspace=torch.empty(sp.host_workspace_min_bytes(), dtype=torch.uint8, device="cuda"))
    torch.cuda.synchronize()
    assert sp.launch_count() == before
    out = torch.full((4,), 3 + 3j, dtype=torch.complex64, device="cuda")
    sp.nudft(torch.rand(4, device="cuda"), e, torch.empty(0, dtype=torch.complex64, device="cuda"), out=out)
    torch.cuda.synchronize()
    assert torch.all(out == 0)
