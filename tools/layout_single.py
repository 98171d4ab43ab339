"""Hot-path GB/s on selected pointer layouts with ONE library loaded in the process (GPU box):
the cross-check of tools/ab_layouts.py, which loads several libraries into one process.

  python tools/layout_single.py LIB.so [CASES]     # CASES: "all" (72 layouts, default) or "hyb"

C2 size, variants N and A, 3 warm-up launches then the median of 7 rounds of 5 launches per
layout.  One JSON line: {"lib": ..., "GBps": {"v0": {...}, "v1": {...}}}."""
import ctypes
import json
import os
import statistics
import sys

import torch

N = 1 << 28


def cases(which):
    out = [(f"sin+{a} cos+{b}", a, b) for a in range(8) for b in range(8)]
    if which == "hyb":
        out = [c for c in out if c[1] and c[2] and c[1] != c[2]] + [("sin+0 cos+0", 0, 0)]
    return out


def main():
    path = os.path.abspath(sys.argv[1])
    which = sys.argv[2] if len(sys.argv) > 2 else "all"
    L = ctypes.CDLL(path)
    L.sincos_pairs.restype = ctypes.c_int
    L.sincos_pairs.argtypes = [ctypes.c_void_p] * 4 + [ctypes.c_size_t, ctypes.c_int, ctypes.c_void_p]
    st = torch.cuda.current_stream().cuda_stream
    tb = torch.rand(N + 16, device="cuda") * 2e4 - 1e4
    sb = torch.empty(N + 16, device="cuda")
    cb = torch.empty(N + 16, device="cuda")
    res = {}
    for v in (0, 1):
        g = {}
        for name, a, b in cases(which):
            def go():
                r = L.sincos_pairs(tb.data_ptr(), sb.data_ptr() + 4 * a, cb.data_ptr() + 4 * b, None, N, v, st)
                assert r == 0, r
            for _ in range(3):
                go()
            ms = []
            for _ in range(7):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(5):
                    go()
                e1.record()
                torch.cuda.synchronize()
                ms.append(e0.elapsed_time(e1) / 5)
            g[name] = round(12 * N / (statistics.median(ms) / 1e3) / 1e9, 1)
        res[f"v{v}"] = g
    print(json.dumps({"lib": os.path.basename(path), "GBps": res}), flush=True)


if __name__ == "__main__":
    main()
