"""A/B of libraries in tools/ab/*.so on the hot path at theta offsets 0 and 4 floats (GPU box).
  python tools/ab_offsets.py"""
import ctypes
import glob
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

n = 1 << 28
base = torch.rand(n + 8, device="cuda") * 2e4 - 1e4
s = torch.empty(n, device="cuda")
c = torch.empty(n, device="cuda")
st = torch.cuda.current_stream().cuda_stream
libs = {}
for p in sorted(glob.glob(os.path.join(ROOT, "tools", "ab", "*.so"))):
    L = ctypes.CDLL(p)
    L.sincos_pairs.restype = ctypes.c_int
    L.sincos_pairs.argtypes = [ctypes.c_void_p] * 4 + [ctypes.c_size_t, ctypes.c_int, ctypes.c_void_p]
    libs[os.path.basename(p)[:-3]] = L
res = {k: {} for k in libs}
for _ in range(3):
    for name, L in libs.items():
        for to in (0, 4, 1):
            th = base[to:to + n]
            fn = lambda: L.sincos_pairs(th.data_ptr(), s.data_ptr(), c.data_ptr(), None, n, 0, st)  # noqa: E731
            for _ in range(2):
                fn()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(10):
                fn()
            b.record()
            torch.cuda.synchronize()
            res[name].setdefault(f"theta+{to}", []).append(12 * n / (a.elapsed_time(b) / 10 / 1e3) / 1e9)
for name in libs:
    print(json.dumps({"lib": name, "GBps": {k: round(statistics.median(v), 1) for k, v in res[name].items()}}))
