"""Cache-policy experiment for the hot kernel's 256-bit loads/stores (GPU box; tuning aid).

Builds variants of libsincos_pairs.so into /tmp with -DSINCOS_LD8_Q / -DSINCOS_ST8_Q and
times the no-math traffic kernel and variant N on the C2 batch (12 B/pair), interleaved over
rounds.  Prints one JSON line per policy pair.   python tools/hint_experiment.py
"""
import ctypes
import itertools
import json
import os
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import inputs  # noqa: E402
from paper_cs_0406049_b200 import _build  # noqa: E402

LOADS = ["", ".L1::no_allocate", ".L1::no_allocate.L2::evict_first", ".L2::evict_last",
         ".L1::no_allocate.L2::evict_normal"]
STORES = ["", ".L1::no_allocate", ".L1::no_allocate.L2::evict_first", ".cs", ".L2::evict_last"]


def build(i, ld, st):
    out = f"/tmp/libsincos_hint{i}.so"
    cmd = [_build.nvcc(), *_build.NVCC_FLAGS, f"-DSINCOS_LD8_Q=\"{ld}\"", f"-DSINCOS_ST8_Q=\"{st}\"", "-o", out,
           *_build.sources()]
    subprocess.check_call(cmd, cwd=_build.PKG)
    L = ctypes.CDLL(out)
    for fn in ("sincos_pairs", "sincos_null_4in8out"):
        getattr(L, fn).restype = ctypes.c_int
    L.sincos_pairs.argtypes = [ctypes.c_void_p] * 4 + [ctypes.c_size_t, ctypes.c_int, ctypes.c_void_p]
    L.sincos_null_4in8out.argtypes = [ctypes.c_void_p] * 4 + [ctypes.c_size_t, ctypes.c_void_p]
    return L


def main():
    n = 1 << 28
    th = torch.from_numpy(inputs.generate(2, 0, n)).cuda()
    s = torch.empty(n, device="cuda")
    c = torch.empty(n, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    combos = [(ld, stq) for ld, stq in itertools.product(LOADS, STORES)
              if not (ld == "" and stq == "")] + [("", "")]
    libs = [build(i, ld, stq) for i, (ld, stq) in enumerate(combos)]
    res = {i: {"null": [], "N": []} for i in range(len(combos))}

    def timeit(fn, reps=10):
        for _ in range(2):
            fn()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            fn()
        b.record()
        torch.cuda.synchronize()
        return 12 * n / (a.elapsed_time(b) / reps / 1e3) / 1e9

    for _ in range(3):
        for i, L in enumerate(libs):
            res[i]["null"].append(timeit(lambda: L.sincos_null_4in8out(th.data_ptr(), s.data_ptr(), c.data_ptr(),
                                                                       None, n, st)))
            res[i]["N"].append(timeit(lambda: L.sincos_pairs(th.data_ptr(), s.data_ptr(), c.data_ptr(), None, n, 0,
                                                             st)))
    for i, (ld, stq) in enumerate(combos):
        print(json.dumps({"load": ld, "store": stq,
                          "GBps": {k: round(statistics.median(v), 1) for k, v in res[i].items()}}), flush=True)


if __name__ == "__main__":
    main()
