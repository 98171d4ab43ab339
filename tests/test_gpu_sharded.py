"""The native single-process multi-device paths on the devices present -- one on
this pool: sincos_pairs_sharded (one host thread per device; forced onto its worker threads
with SINCOS_SHARDED_WORKERS=1 so one GPU exercises them) and sincos_pairs_sharded_stats (a
1-rank NCCL communicator still runs ncclCommInitAll and ncclAllGather), their validation before
any launch, error codes, and the communicator kept across calls.  ``pytest -m gpu``."""
import os
import subprocess
import sys
import textwrap
import time

import numpy as np
import pytest

import inputs
import oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_cs_0406049_b200 as sp  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OK, INVALID, OVERLAP, CUDA, NCCL = 0, 1, 2, 3, 4


@pytest.fixture(scope="module", autouse=True)
def cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    yield


def make_shards(n, G_dev, inter, per_device=1, seed=5):
    th_all = inputs.generate(seed, 0, n)
    shards = []
    G = G_dev * per_device
    for g in range(G):
        lo, hi = sp.shard_range(n, G, g)
        dev = torch.device("cuda", g % G_dev)
        t = torch.from_numpy(th_all[lo:hi]).to(dev)
        sh = {"theta": t}
        if inter:
            sh["inter"] = torch.empty(2 * (hi - lo), device=dev)
        else:
            sh["sin"], sh["cos"] = torch.empty_like(t), torch.empty_like(t)
        shards.append(sh)
    return th_all, shards


@pytest.mark.parametrize("variant", [0, 1])
@pytest.mark.parametrize("inter", [False, True])
def test_sharded_stats_on_available_devices(variant, inter):
    G = torch.cuda.device_count()
    _, shards = make_shards((1 << 22) + 5, G, inter)
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


_REUSE_SCRIPT = textwrap.dedent("""
    import sys, time, torch
    sys.path.insert(0, {root!r})
    import inputs, paper_cs_0406049_b200 as sp
    G = torch.cuda.device_count()
    t = [torch.from_numpy(inputs.generate(2, 0, 1 << 20)).to(f"cuda:{{g}}") for g in range(G)]
    shards = [{{"theta": x, "sin": torch.empty_like(x), "cos": torch.empty_like(x)}} for x in t]
    keys = ("n", "nan_count", "max_comb", "sum_sq", "max_amp", "worst_theta", "device")
    times, recs = [], []
    for _ in range(4):
        t0 = time.perf_counter()
        r = sp.sincos_pairs_sharded_stats(shards)
        times.append(time.perf_counter() - t0)
        recs.append([[x[k] for k in keys] for x in r])
    assert all(r == recs[0] for r in recs), recs
    print("times", times)
    assert max(times[1:]) < 0.5 * times[0], times
    print("reuse ok")
""")


def test_sharded_stats_reuses_its_communicator():
    """The communicator and buffers are created once per device list: in a fresh process the
    first call pays ncclCommInitAll, later calls on the same devices reuse it (much faster) and
    return the same records."""
    r = subprocess.run([sys.executable, "-c", _REUSE_SCRIPT.format(root=ROOT)], capture_output=True, text=True,
                       timeout=600, cwd=ROOT)
    assert r.returncode == 0 and "reuse ok" in r.stdout, (r.stdout[-2000:], r.stderr[-3000:])


def test_sharded_stats_validation_and_errors():
    """Refused before anything is launched: a device ordinal past the device count, two
    shards on one device, a bad variant; nothing launched, outputs untouched."""
    L = sp.lib()
    _, shards = make_shards(1 << 16, 1, False)
    arr = sp._shard_array(shards)
    out = (sp.Stats * 1)()
    shards[0]["sin"].fill_(7.0)
    before = sp.launch_count()
    arr[0].device = torch.cuda.device_count() + 3
    assert L.sincos_pairs_sharded_stats(arr, 1, 0, out) == INVALID
    arr[0].device = -1
    assert L.sincos_pairs_sharded_stats(arr, 1, 0, out) == INVALID
    arr[0].device = 0
    assert L.sincos_pairs_sharded_stats(arr, 1, 5, out) == INVALID
    arr2 = (sp.Shard * 2)(arr[0], arr[0])
    assert L.sincos_pairs_sharded_stats(arr2, 2, 0, (sp.Stats * 2)()) == INVALID
    torch.cuda.synchronize()
    assert sp.launch_count() == before and bool((shards[0]["sin"] == 7.0).all())
    assert L.sincos_status_string(NCCL) and L.sincos_last_nccl_error() == 0


@pytest.mark.parametrize("inter", [False, True])
def test_sharded_validation_before_any_launch(inter):
    """sincos_pairs_sharded checks every shard -- buffers and device ordinals -- before it
    launches any: a bad pointer or device in the middle of the list leaves every output
    untouched and the launch count unchanged."""
    L = sp.lib()
    _, shards = make_shards((1 << 18) + 3, 1, inter, per_device=4)
    for sh in shards:
        for k in ("sin", "cos", "inter"):
            if k in sh:
                sh[k].fill_(7.0)
    torch.cuda.synchronize()
    before = sp.launch_count()
    arr = sp._shard_array(shards)
    arr[2].theta_dev = arr[2].theta_dev + 2                 # 2-B aligned theta in shard 2
    assert L.sincos_pairs_sharded(arr, 4, 0) == INVALID
    arr = sp._shard_array(shards)
    arr[2].device = torch.cuda.device_count() + 5           # no such device
    assert L.sincos_pairs_sharded(arr, 4, 0) == INVALID
    arr = sp._shard_array(shards)
    if inter:
        arr[3].inter_dev = arr[3].theta_dev                 # theta inside its interleaved output
    else:
        arr[3].cos_dev = arr[3].sin_dev + 4                 # sin and cos overlap
    assert L.sincos_pairs_sharded(arr, 4, 0) == OVERLAP
    arr = sp._shard_array(shards)
    assert L.sincos_pairs_sharded(arr, 4, 9) == INVALID     # variant
    torch.cuda.synchronize()
    assert sp.launch_count() == before
    for sh in shards:
        for k in ("sin", "cos", "inter"):
            if k in sh:
                assert bool((sh[k] == 7.0).all()), k
    assert L.sincos_pairs_sharded(arr, 0, 0) == OK           # empty list


_WORKER_SCRIPT = textwrap.dedent("""
    import sys, numpy as np, torch
    sys.path.insert(0, {root!r})
    import inputs, oracle, paper_cs_0406049_b200 as sp
    n = (1 << 22) + 13
    th = inputs.generate(5, 0, n)
    for inter in (False, True):
        for v in (0, 1):
            G = 8
            shards = []
            for g in range(G):
                lo, hi = sp.shard_range(n, G, g)
                t = torch.from_numpy(th[lo:hi]).cuda()
                sh = {{"theta": t, "stream": torch.cuda.Stream() if g % 2 else None}}
                if inter:
                    sh["inter"] = torch.empty(2 * (hi - lo), device="cuda")
                else:
                    sh["sin"], sh["cos"] = torch.empty_like(t), torch.empty_like(t)
                shards.append(sh)
            before = sp.launch_count()
            sp.sincos_pairs_sharded(shards, variant=v)
            torch.cuda.synchronize()
            assert sp.launch_count() - before == G
            if inter:
                o = torch.cat([sh["inter"] for sh in shards]).cpu().numpy()
                s, c = o[1::2], o[0::2]
            else:
                s = torch.cat([sh["sin"] for sh in shards]).cpu().numpy()
                c = torch.cat([sh["cos"] for sh in shards]).cpu().numpy()
            ws, wc = oracle.sincos(th, v)
            assert np.array_equal(s, ws) and np.array_equal(c, wc), (inter, v)
            assert torch.cuda.current_device() == 0
    # concurrent callers share the worker: both complete, both correct
    import threading
    res = []
    def call():
        t = torch.from_numpy(th).cuda(); s = torch.empty_like(t); c = torch.empty_like(t)
        sp.sincos_pairs_sharded([{{"theta": t, "sin": s, "cos": c}}])
        torch.cuda.synchronize()
        res.append(np.array_equal(s.cpu().numpy(), oracle.sincos(th, 0)[0]))
    ts = [threading.Thread(target=call) for _ in range(4)]
    [t.start() for t in ts]; [t.join() for t in ts]
    assert res == [True] * 4, res
    print("workers ok")
""")


def test_sharded_through_worker_threads():
    """The one-host-thread-per-device launch machinery, forced on for one device
    (SINCOS_SHARDED_WORKERS=1): 8 shards (some on side streams) through the device's worker,
    bit-identical to the oracle, the caller's current device unchanged; concurrent callers."""
    env = dict(os.environ, SINCOS_SHARDED_WORKERS="1")
    r = subprocess.run([sys.executable, "-c", _WORKER_SCRIPT.format(root=ROOT)], capture_output=True, text=True,
                       timeout=600, env=env, cwd=ROOT)
    assert r.returncode == 0 and "workers ok" in r.stdout, r.stderr[-3000:]
