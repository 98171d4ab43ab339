"""The native single-process sharded run with NCCL-gathered statistics
(sincos_pairs_sharded_stats) on the devices present (one on this pool: a 1-rank NCCL
communicator still runs ncclCommInitAll and ncclAllGather).  ``pytest -m gpu``."""
import numpy as np
import pytest

import inputs
import oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_cs_0406049_b200 as sp  # noqa: E402


@pytest.mark.parametrize("variant", [0, 1])
@pytest.mark.parametrize("inter", [False, True])
def test_sharded_stats_on_available_devices(variant, inter):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    G = torch.cuda.device_count()
    n = (1 << 22) + 5
    th_all = inputs.generate(5, 0, n)
    shards = []
    for g in range(G):
        lo, hi = sp.shard_range(n, G, g)
        dev = torch.device("cuda", g)
        t = torch.from_numpy(th_all[lo:hi]).to(dev)
        sh = {"theta": t}
        if inter:
            sh["inter"] = torch.empty(2 * (hi - lo), device=dev)
        else:
            sh["sin"], sh["cos"] = torch.empty_like(t), torch.empty_like(t)
        shards.append(sh)
    recs = sp.sincos_pairs_sharded_stats(shards, variant=variant)
    assert len(recs) == G
    for g, (sh, r) in enumerate(zip(shards, recs)):
        ref = sp.error_stats(sh["theta"], sh.get("sin"), sh.get("cos"), sh.get("inter"))
        for k in ("n", "nan_count", "max_comb", "sum_sq", "max_amp", "worst_theta"):
            assert r[k] == ref[k], k
        assert r["device"] == g and r["kernel_ms"] > 0
        # and the shard's outputs are the oracle's
        th = sh["theta"].cpu().numpy()
        ws, wc = oracle.sincos(th[:100000], variant)
        if inter:
            o = sh["inter"].cpu().numpy()[:200000]
            s, c = o[1::2], o[0::2]
        else:
            s, c = sh["sin"].cpu().numpy()[:100000], sh["cos"].cpu().numpy()[:100000]
        assert np.array_equal(s, ws) and np.array_equal(c, wc)
