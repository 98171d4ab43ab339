"""16-bit split outputs with cos[] at every element offset 0..7 from sin[]'s 16-B frame (GPU box):
GB/s (8 B per pair) of sincos_pairs_dtype at the C2 size for fp16 / bf16, variants N and A --
the product (cos[] piece stores) beside the one-element-per-thread path (A/B build,
realign = 0), which these layouts took before; then the general-method path (fp32, 12 B per pair)
with cos[] at every float offset from sin[]'s 32-B frame.  3 warm-up launches, median of 5 rounds x 5.
  python tools/dtype_offsets_probe.py"""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_cs_0406049_b200 as sp  # noqa: E402
from paper_cs_0406049_b200 import ab  # noqa: E402

N = 1 << 28


def timed(fn):
    for _ in range(3):
        fn()
    ms = []
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(5):
            fn()
        b.record()
        torch.cuda.synchronize()
        ms.append(a.elapsed_time(b) / 5)
    return round(8 * N / (statistics.median(ms) / 1e3) / 1e9, 1)


def main():
    t = torch.rand(N, device="cuda") * 2e4 - 1e4
    res = {}
    for dt, dname in ((torch.float16, "fp16"), (torch.bfloat16, "bf16")):
        sb = torch.empty(N + 16, dtype=dt, device="cuda")
        cb = torch.empty(N + 16, dtype=dt, device="cuda")
        for v in (0, 1):
            for oc in range(8):
                s, c = sb[:N], cb[oc:oc + N]
                key = f"{dname}_{'NA'[v]}_cos+{oc}"
                res[key] = {"product": timed(lambda: sp.sincos_pairs_dtype(t, s, c, variant=v))}
                with ab.knobs(realign=0):
                    res[key]["one_per_thread"] = timed(lambda: sp.sincos_pairs_dtype(t, s, c, variant=v))
                print(json.dumps({key: res[key]}), flush=True)
    # the general method (paper's table N), fp32 split outputs, cos[] at float offsets 0..7
    m = sp.make_method(*sp.PAPER_METHODS[0])
    sb = torch.empty(N + 16, device="cuda")
    cb = torch.empty(N + 16, device="cuda")
    for oc in range(8):
        s, c = sb[:N], cb[oc:oc + N]
        key = f"method_N_cos+{oc}"
        res[key] = {"product": round(timed(lambda: sp.sincos_pairs_method(t, m, s, c)) * 1.5, 1)}
        with ab.knobs(realign=0):
            res[key]["one_per_thread"] = round(timed(lambda: sp.sincos_pairs_method(t, m, s, c)) * 1.5, 1)
        print(json.dumps({key: res[key]}), flush=True)
    ib = torch.empty(2 * N + 16, device="cuda")
    for oi in range(8):                               # interleaved pairs at float offsets 0..7
        io = ib[oi:oi + 2 * N]
        key = f"method_N_inter+{oi}"
        res[key] = {"product": round(timed(lambda: sp.sincos_pairs_method(t, m, interleaved_out=io)) * 1.5, 1)}
        with ab.knobs(realign=0):
            res[key]["one_per_thread"] = round(
                timed(lambda: sp.sincos_pairs_method(t, m, interleaved_out=io)) * 1.5, 1)
        print(json.dumps({key: res[key]}), flush=True)


if __name__ == "__main__":
    main()
