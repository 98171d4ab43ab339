"""The N>1 host path on CPU: world_size-2 gloo process group (prompt item 5).

Covers what a multi-GPU bench run does besides the kernel: each rank takes its contiguous
shard from the C-ABI sharder, computes it (here with the oracle, standing in for the GPU
kernel, whose parity is tested separately), gathers the per-shard statistics records over
the process group, takes the max of the per-rank times, and rank 0 aggregates.  The
concatenated shards must equal the whole-array computation bit for bit."""
import os
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import inputs
import oracle
from paper_cs_0406049_b200.sharding import WORKLOADS, gather_records, max_over_ranks, summarize


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, outdir, wname):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        W = WORKLOADS[wname]
        lo, hi = W.rank_range(world, rank)
        th = inputs.generate(W.config, lo, hi - lo)
        recs = []
        for v in (oracle.VARIANT_N, oracle.VARIANT_A):
            s, c = oracle.sincos(th, v)
            np.save(os.path.join(outdir, f"r{rank}_v{v}_s.npy"), s)
            np.save(os.path.join(outdir, f"r{rank}_v{v}_c.npy"), c)
            st = oracle.error_stats(th, s, c)
            recs.append([float(st.count), float(st.nan_count), st.max_comb, st.sum_sq, st.max_amp,
                         1.0 + rank, float(rank), float(v)])
        allrecs = gather_records(recs, world)
        tmax = max_over_ranks(1.0 + rank, world)
        if rank == 0:
            summ = summarize(allrecs)
            np.save(os.path.join(outdir, "summary.npy"),
                    np.array([summ["n"], summ["max_err"], summ["rms_err"], summ["nan"], tmax,
                              summ["slowest_kernel_ms"], len(summ["shards"])], dtype=np.float64))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("wname", ["c1", "c3"])
def test_two_rank_gloo_shards_and_stats(wname):
    world = 2
    W = WORKLOADS[wname]
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(world, _free_port(), d, wname), nprocs=world, join=True)
        th = inputs.generate(W.config, 0, W.n)
        for v in (oracle.VARIANT_N, oracle.VARIANT_A):
            s = np.concatenate([np.load(os.path.join(d, f"r{r}_v{v}_s.npy")) for r in range(world)])
            c = np.concatenate([np.load(os.path.join(d, f"r{r}_v{v}_c.npy")) for r in range(world)])
            ws, wc = oracle.sincos(th, v)
            assert s.size == W.n
            assert np.array_equal(s.view(np.uint32), ws.view(np.uint32))
            assert np.array_equal(c.view(np.uint32), wc.view(np.uint32))
        summ = np.load(os.path.join(d, "summary.npy"))
        n_fin = np.count_nonzero(np.isfinite(th))
        assert summ[0] == 2 * n_fin                   # both variants' finite elements
        st = oracle.error_stats(th, *oracle.sincos(th, oracle.VARIANT_N))
        sa = oracle.error_stats(th, *oracle.sincos(th, oracle.VARIANT_A))
        assert summ[1] == max(st.max_comb, sa.max_comb)
        assert abs(summ[2] / np.sqrt((st.sum_sq + sa.sum_sq) / (st.count + sa.count)) - 1) < 1e-9   # summation order
        assert summ[4] == 2.0 and summ[5] == 2.0 and summ[6] == 2 * world


def test_weak_and_strong_rank_ranges():
    """c2 is weak scaling (each rank a fresh 2^28 slice of the stream); c4/c5 are contiguous
    shards of the fixed array, row blocks for c4."""
    c2, c4, c5 = WORKLOADS["c2"], WORKLOADS["c4"], WORKLOADS["c5"]
    assert [c2.rank_range(4, r) for r in range(4)] == [(r << 28, (r + 1) << 28) for r in range(4)]
    for G in (1, 2, 4, 8):
        rr = [c4.rank_range(G, r) for r in range(G)]
        assert rr[0][0] == 0 and rr[-1][1] == 1 << 30
        assert all(lo % (1 << 15) == 0 for lo, _ in rr)      # whole rows of 2^15 phases
        rr = [c5.rank_range(G, r) for r in range(G)]
        assert sum(hi - lo for lo, hi in rr) == 1 << 32
