"""Host-side cost per call of the Python binding on a tiny array (GPU box): the ctypes call
alone vs sincos_pairs() vs sincos() (allocating).  python tools/binding_overhead.py"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_cs_0406049_b200 as sp  # noqa: E402


def per_call(fn, k=5000):
    for _ in range(100):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(k):
        fn()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    return 1e6 * (t1 - t0) / k


def main():
    t = torch.rand(1024, device="cuda")
    s, c = torch.empty_like(t), torch.empty_like(t)
    L = sp.lib()
    st = torch.cuda.current_stream().cuda_stream
    tp, spp, cp = t.data_ptr(), s.data_ptr(), c.data_ptr()
    out = {"raw_ctypes_us": per_call(lambda: L.sincos_pairs(tp, spp, cp, None, 1024, 0, st)),
           "sincos_pairs_us": per_call(lambda: sp.sincos_pairs(t, s, c)),
           "sincos_alloc_us": per_call(lambda: sp.sincos(t))}
    print(json.dumps({k: round(v, 2) for k, v in out.items()}))


if __name__ == "__main__":
    main()
