"""Per-GPU shard times for G = 1, 2, 4, 8 on ONE B200 (projection aid; GPU box).

The path shards with no exchange step: at G GPUs each rank runs the same
kernel on its own contiguous shard, so the job time is the slowest rank's kernel time.  On a
one-GPU box this tool times the kernel on every shard size the sharder produces for G GPUs
(shard 0 of sincos_shard_range, device-resident, event-timed, both variants), and reports
the projected aggregate pairs/s = n_total / t_shard.  A projection, not a multi-GPU
measurement: it leaves out launch skew between processes (none: one process per GPU) and any
NVLink/NVSwitch effect (none: no data crosses devices).
  python tools/shard_projection.py  ->  one JSON line per workload"""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import inputs  # noqa: E402
import paper_cs_0406049_b200 as sp  # noqa: E402
from paper_cs_0406049_b200.sharding import WORKLOADS  # noqa: E402


def time_kernel(th, outs, v, reps):
    """Median per-launch time of `reps` back-to-back launches (events between consecutive
    launches on the stream, no host sync in between -- as bench.py times its steps)."""
    for _ in range(3):
        sp.sincos_pairs(th, variant=v, **outs)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(reps + 1)]
    ev[0].record()
    for k in range(reps):
        sp.sincos_pairs(th, variant=v, **outs)
        ev[k + 1].record()
    torch.cuda.synchronize()
    return statistics.median(ev[k].elapsed_time(ev[k + 1]) for k in range(reps))


def main():
    for wname in ("c2", "c4", "c5"):
        W = WORKLOADS[wname]
        res = {"workload": W.description, "scaling": "weak" if W.weak else "strong", "per_G": {}}
        n_max = W.n if not W.weak else W.n
        th_all = torch.empty(n_max, dtype=torch.float32, device="cuda")
        chunk = 1 << 28
        for off in range(0, n_max, chunk):
            m = min(chunk, n_max - off)
            th_all[off:off + m].copy_(torch.from_numpy(inputs.generate(W.config, off, m)))
        if W.interleaved:
            out_all = {"interleaved_out": torch.empty(2 * n_max, dtype=torch.float32, device="cuda")}
        else:
            out_all = {"sin_out": torch.empty(n_max, dtype=torch.float32, device="cuda"),
                       "cos_out": torch.empty(n_max, dtype=torch.float32, device="cuda")}
        for G in (1, 2, 4, 8):
            lo, hi = W.rank_range(G, 0)
            n = hi - lo
            th = th_all[:n]
            outs = {k: v[:2 * n] if k == "interleaved_out" else v[:n] for k, v in out_all.items()}
            t = {vn: time_kernel(th, outs, v, 20 if n >= (1 << 28) else 50)
                 for vn, v in (("N", sp.NORMALIZED), ("A", sp.RENORMALIZED))}
            step_ms = t["N"] + t["A"]
            total = n * G if W.weak else W.n
            res["per_G"][G] = {"shard_elements": n, "kernel_ms": t, "GBps_per_gpu": {k: 12 * n / (x / 1e3) / 1e9
                                                                                    for k, x in t.items()},
                               "projected_pairs_per_s": 2 * total / (step_ms / 1e3)}
        base = res["per_G"][1]["projected_pairs_per_s"]
        for G in (2, 4, 8):
            res["per_G"][G]["projected_efficiency"] = res["per_G"][G]["projected_pairs_per_s"] / (G * base)
        print(json.dumps(res), flush=True)
        del th_all, out_all
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
