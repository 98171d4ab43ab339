"""Launch-configuration sweep for the hot kernel (tuning aid, GPU only).

Times every candidate (threads, blocks_per_sm, vec, unroll, prefetch) for both variants
and the traffic-ceiling kernel on the C2 workload (2^28 elements, split outputs), in
several interleaved rounds so that clock/DRAM drift spreads over all candidates, and
prints one JSON line per candidate with the median GB/s (12 B per pair).

  python tools/sweep_launch.py [--n 268435456] [--rounds 3] [--reps 10] [--inter]
"""
import argparse
import itertools
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import inputs  # noqa: E402
import paper_cs_0406049_b200 as sp  # noqa: E402
from paper_cs_0406049_b200 import ab  # A/B build (tools only)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1 << 28)
    ap.add_argument("--rounds", type=int, default=3)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--inter", action="store_true")
    ap.add_argument("--threads", default="128,256,512")
    ap.add_argument("--bps", default="0,8,16,32,4096")
    ap.add_argument("--vec", default="8")
    ap.add_argument("--unroll", default="1,2,4")
    ap.add_argument("--prefetch", default="0,1")
    args = ap.parse_args()
    n = args.n
    th = torch.from_numpy(inputs.generate(2, 0, n)).cuda()
    if args.inter:
        outs = dict(interleaved_out=torch.empty(2 * n, device="cuda"))
    else:
        outs = dict(sin_out=torch.empty(n, device="cuda"), cos_out=torch.empty(n, device="cuda"))
    ints = lambda s: [int(x) for x in s.split(",")]  # noqa: E731
    cands = list(itertools.product(ints(args.threads), ints(args.bps), ints(args.vec), ints(args.unroll),
                                   ints(args.prefetch)))
    res = {c: {"N": [], "A": [], "null": []} for c in cands}
    stream = torch.cuda.current_stream()

    def timeit(fn):
        for _ in range(2):
            fn()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(args.reps):
            fn()
        b.record(stream)
        torch.cuda.synchronize()
        return 12 * n / (a.elapsed_time(b) / args.reps / 1e3) / 1e9

    for _ in range(args.rounds):
        for c in cands:
            ab.set_launch_config(*c)
            res[c]["N"].append(timeit(lambda: sp.sincos_pairs(th, variant=0, **outs)))
            res[c]["A"].append(timeit(lambda: sp.sincos_pairs(th, variant=1, **outs)))
            res[c]["null"].append(timeit(lambda: sp.null_4in8out(th, **outs)))
    for c in cands:
        med = {k: round(statistics.median(v), 1) for k, v in res[c].items()}
        spread = {k: round(max(v) - min(v), 1) for k, v in res[c].items()}
        print(json.dumps({"cfg": dict(zip(("threads", "bps", "vec", "unroll", "prefetch"), c)),
                          "GBps": med, "spread": spread, "inter": args.inter}), flush=True)


if __name__ == "__main__":
    main()
