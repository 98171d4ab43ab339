"""sincos_pairs_batched of the A/B build (outside SURVEY 8, not in the product library): many
arrays in one launch (per 480), each bit-exact vs the oracle.  ``pytest -m gpu``."""
import numpy as np
import pytest

import inputs
import oracle
from helpers import assert_parity

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_cs_0406049_b200 as sp  # noqa: E402
from paper_cs_0406049_b200 import ab  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    yield


@pytest.mark.parametrize("count", [1, 7, 480, 481, 1000])
@pytest.mark.parametrize("inter", [False, True])
@pytest.mark.parametrize("variant", [0, 1])
def test_batched_matches_oracle(count, inter, variant):
    """Random lengths (0 .. ~5000, some past one 1024-element chunk), random theta/output
    offsets (vector and one-per-thread items mixed), some exact in-place items (split);
    counts across the 480-item launch boundary."""
    rng = np.random.default_rng(count * 4 + 2 * inter + variant)
    lens = rng.integers(0, 5000, count)
    lens[rng.random(count) < 0.1] = 0
    base = torch.from_numpy(inputs.generate(3, 0, int(lens.sum()) + 16 * count)).cuda()
    thetas, outs_s, outs_c, outs_i, wants = [], [], [], [], []
    off = 0
    for i, n in enumerate(lens):
        n = int(n)
        ot = int(rng.integers(0, 8))
        th = base[off + ot:off + ot + n]
        off += n + 16
        ws, wc = oracle.sincos(th.cpu().numpy(), variant)
        wants.append((ws, wc))
        if inter:
            oo = int(rng.integers(0, 8))
            outs_i.append(torch.empty(2 * n + 8, device="cuda")[oo:oo + 2 * n])
        elif rng.random() < 0.1 and n > 0:
            th = th.clone()                                   # exact in place: sin over theta
            outs_s.append(th)
            outs_c.append(torch.empty(n, device="cuda"))
        else:
            oo = int(rng.integers(0, 8))
            outs_s.append(torch.empty(n + 8, device="cuda")[oo:oo + n])
            outs_c.append(torch.empty(n + 8, device="cuda")[oo:oo + n])
        thetas.append(th)
    if inter:
        ab.sincos_pairs_batched(thetas, interleaved_outs=outs_i, variant=variant)
    else:
        ab.sincos_pairs_batched(thetas, outs_s, outs_c, variant=variant)
    torch.cuda.synchronize()
    for i, (ws, wc) in enumerate(wants):
        if inter:
            o = outs_i[i].cpu().numpy()
            assert_parity(o[1::2], o[0::2], ws, wc, f"item {i} n={lens[i]}")
        else:
            assert_parity(outs_s[i].cpu().numpy(), outs_c[i].cpu().numpy(), ws, wc, f"item {i} n={lens[i]}")


def test_batched_list_form_and_validation():
    ts = [torch.rand(n, device="cuda") * 10 for n in (5, 1000, 3000)]
    ss, cs = [torch.empty_like(t) for t in ts], [torch.empty_like(t) for t in ts]
    ab.sincos_pairs_batched(ts, ss, cs)
    for t, s, c in zip(ts, ss, cs):
        ws, wc = oracle.sincos(t.cpu().numpy(), 0)
        assert_parity(s.cpu().numpy(), c.cpu().numpy(), ws, wc, "list form")
    ab.sincos_pairs_batched([])                               # empty batch: no-op
    t = torch.rand(64, device="cuda")
    s = torch.empty(64, device="cuda")
    with pytest.raises(sp.SincosError):                       # overlap inside an item: refused
        ab.sincos_pairs_batched([t], [s], [s])
