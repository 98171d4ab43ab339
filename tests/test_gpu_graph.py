"""The C-ABI launches are capturable in a CUDA graph (used by bench.py for the launch-bound
small configs) and replay bit-identically.  ``pytest -m gpu``."""
import pytest

import inputs

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_cs_0406049_b200 as sp  # noqa: E402


@pytest.mark.parametrize("variant", [0, 1])
def test_graph_capture_and_replay(variant):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    t = torch.from_numpy(inputs.generate(1)).cuda()
    s0, c0 = sp.sincos(t, variant=variant)
    s, c = torch.zeros_like(t), torch.zeros_like(t)
    o = torch.zeros(2 * t.numel(), device="cuda")
    g = torch.cuda.CUDAGraph()
    cap = torch.cuda.Stream()
    cap.wait_stream(torch.cuda.current_stream())
    with torch.cuda.graph(g, stream=cap):
        sp.sincos_pairs(t, s, c, variant=variant, stream=cap)
        sp.sincos_pairs(t, interleaved_out=o, variant=variant, stream=cap)
    torch.cuda.synchronize()
    for _ in range(3):
        s.zero_()
        o.zero_()
        g.replay()
        torch.cuda.synchronize()
        assert torch.equal(s, s0) and torch.equal(c, c0)
        assert torch.equal(o[1::2], s0) and torch.equal(o[0::2], c0)
