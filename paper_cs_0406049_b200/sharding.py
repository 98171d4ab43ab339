"""Host-side sharding and the per-shard statistics exchange.

The path is embarrassingly parallel (every element independent), so a
multi-GPU run shards the array into contiguous ranges, one per rank (one process
per GPU), with no data-path collective.  The only collective is the gather of a
small per-shard record (error statistics and kernel time) after the timed region
-- NCCL on GPUs, gloo in the CPU tests.  Shard boundaries come from the C ABI's
sincos_shard_range (8-element aligned starts).
"""
from __future__ import annotations

from dataclasses import dataclass

from . import shard_range

# the gathered record: n, nan_count, max_err, sum_sq_err, max_amp, kernel_ms, rank, variant
RECORD_FIELDS = ("n", "nan_count", "max_err", "sum_sq", "max_amp", "kernel_ms", "rank", "variant")


@dataclass(frozen=True)
class Workload:
    """One BASELINE.json config as a bench workload."""
    name: str
    config: int          # inputs.generate config id
    n: int               # elements: per rank (weak) or in total (strong)
    interleaved: bool
    weak: bool
    description: str

    def rank_range(self, world: int, rank: int):
        """[lo, hi) of this rank's elements in the config's counter stream."""
        if self.weak:
            return rank * self.n, (rank + 1) * self.n
        return shard_range(self.n, world, rank)


WORKLOADS = {
    "c1": Workload("c1", 1, 1 << 20, False, False, "C1: 2^20 U[-pi,pi) seed 0, split, contiguous shards"),
    "c2": Workload("c2", 2, 1 << 28, False, True,
                   "C2: 2^28 fp32 angles U[-1e4,1e4] seed 1 per GPU, split sin/cos, both variants (N then A) per step"),
    "c3": Workload("c3", 3, 1 << 24, True, False, "C3: 2^24 edge/stress set seed 2, interleaved, contiguous shards"),
    "c4": Workload("c4", 4, 1 << 30, True, False,
                   "C4: 2^30 NUFFT phases 2pi f_i t_j seed 3, interleaved, sharded by row blocks"),
    "c5": Workload("c5", 5, 1 << 32, False, False,
                   "C5: 2^32 N(0,100^2) seed 4, split, contiguous shards"),
}


def gather_records(records, world: int, device=None):
    """All-gather each rank's list of per-shard records (lists of floats, RECORD_FIELDS order)
    over the default process group; returns the list of all ranks' records (rank order).
    Uses whatever backend the group has (NCCL with CUDA tensors, gloo with CPU ones)."""
    import torch
    import torch.distributed as dist
    mine = torch.tensor(records, dtype=torch.float64, device=device)
    if world == 1:
        return [list(map(float, r)) for r in mine.cpu().tolist()]
    out = [torch.empty_like(mine) for _ in range(world)]
    dist.all_gather(out, mine)
    return [list(map(float, r)) for t in out for r in t.cpu().tolist()]


def max_over_ranks(value: float, world: int, device=None) -> float:
    """The max over ranks of a per-rank time (the timing rule: the job ends with its slowest rank)."""
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def summarize(records):
    """Aggregate gathered per-shard records: overall max error, rms, NaN count, the slowest shard."""
    recs = [dict(zip(RECORD_FIELDS, r)) for r in records]
    n = sum(r["n"] for r in recs)
    out = {
        "shards": [{"rank": int(r["rank"]), "variant": "N" if r["variant"] == 0 else "A", "n": int(r["n"]),
                    "nan": int(r["nan_count"]), "max_err": r["max_err"],
                    "rms_err": (r["sum_sq"] / r["n"]) ** 0.5 if r["n"] else 0.0, "max_amp": r["max_amp"],
                    "kernel_ms": r["kernel_ms"]} for r in recs],
        "n": int(n),
        "max_err": max((r["max_err"] for r in recs), default=0.0),
        "rms_err": (sum(r["sum_sq"] for r in recs) / n) ** 0.5 if n else 0.0,
        "nan": int(sum(r["nan_count"] for r in recs)),
        "slowest_kernel_ms": max((r["kernel_ms"] for r in recs), default=0.0),
    }
    return out
