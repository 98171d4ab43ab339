"""A/B of libraries on the NEXT(4) layout adapters (tuning aid; GPU box): sincos_interleave and
sincos_deinterleave at 2^28 elements (16 B per element: 8 read, 8 written), every
tools/ab_adapters/*.so, median of 5 rounds x 10 launches, libraries interleaved over rounds."""
import ctypes
import glob
import json
import os
import statistics

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    import torch
    libs = {}
    for p in sorted(glob.glob(os.path.join(ROOT, "tools", "ab_adapters", "*.so"))):
        L = ctypes.CDLL(p)
        for fn in (L.sincos_interleave, L.sincos_deinterleave):
            fn.restype = ctypes.c_int
            fn.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_size_t, ctypes.c_void_p]
        libs[os.path.basename(p)[:-3]] = L
    n = 1 << 28
    s, c = torch.rand(n, device="cuda"), torch.rand(n, device="cuda")
    io = torch.empty(2 * n, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    res = {k: {"interleave": [], "deinterleave": []} for k in libs}
    order = list(libs)
    for rnd in range(len(order) * -(-5 // len(order))):   # rotating order (see ab_phase.py)
        for name in order[rnd % len(order):] + order[:rnd % len(order)]:
            L = libs[name]
            for which, call in (("interleave", lambda: L.sincos_interleave(s.data_ptr(), c.data_ptr(), io.data_ptr(), n, st)),
                                ("deinterleave", lambda: L.sincos_deinterleave(io.data_ptr(), s.data_ptr(), c.data_ptr(), n, st))):
                assert call() == 0
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                for _ in range(10):
                    call()
                b.record()
                torch.cuda.synchronize()
                res[name][which].append(16 * n / (a.elapsed_time(b) / 10 / 1e3) / 1e9)
    for name in libs:
        print(json.dumps({"lib": name, **{k: round(statistics.median(v), 1) for k, v in res[name].items()}}))


if __name__ == "__main__":
    main()
