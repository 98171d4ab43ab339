"""Many small arrays: one sincos_pairs_batched call vs one sincos_pairs launch per array
(through ctypes, no Python binding overhead) vs the same per-array launches in a CUDA graph
(GPU box).  Pairs/s over the whole batch.   python tools/batched_probe.py"""
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_cs_0406049_b200 as sp  # noqa: E402
from paper_cs_0406049_b200 import ab  # A/B build (tools only)


def timed(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def main():
    L = ab.lib()
    out = {}
    for count, n in ((1000, 256), (1000, 4096), (100, 65536), (2000, 1000), (10, 4096), (60, 4096)):
        base = torch.rand(count * n, device="cuda") * 200 - 100
        s = torch.empty_like(base)
        c = torch.empty_like(base)
        thetas = [base[i * n:(i + 1) * n] for i in range(count)]
        ss = [s[i * n:(i + 1) * n] for i in range(count)]
        cs = [c[i * n:(i + 1) * n] for i in range(count)]
        st = torch.cuda.current_stream().cuda_stream
        ptrs = [(t.data_ptr(), a.data_ptr(), b.data_ptr()) for t, a, b in zip(thetas, ss, cs)]

        def loop():
            for tp, sp_, cp in ptrs:
                L.sincos_pairs(tp, sp_, cp, None, n, 0, st)

        arr = (ab.Item * count)(*[ab.Item(tp, sp_, cp, None, n) for tp, sp_, cp in ptrs])

        def batched():
            L.sincos_pairs_batched(ctypes.addressof(arr), count, 0, st)

        ms_loop = timed(loop, 5)
        ms_b = timed(batched)
        cap = torch.cuda.Stream()
        cap.wait_stream(torch.cuda.current_stream())
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=cap):
            for tp, sp_, cp in ptrs:
                L.sincos_pairs(tp, sp_, cp, None, n, 0, cap.cuda_stream)
        torch.cuda.current_stream().wait_stream(cap)
        ms_g = timed(g.replay)
        pairs = count * n
        out[f"{count}x{n}"] = {"per_array_launches_ms": round(ms_loop, 3), "graph_of_launches_ms": round(ms_g, 3),
                               "batched_ms": round(ms_b, 4), "batched_G_pairs_per_s": round(pairs / ms_b / 1e6, 1),
                               "speedup_vs_launches": round(ms_loop / ms_b, 1),
                               "speedup_vs_graph": round(ms_g / ms_b, 1)}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
