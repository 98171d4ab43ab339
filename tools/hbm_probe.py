"""HBM traffic-mix probe (context for the roofline; GPU only).

Measures, on 1 GiB-scale buffers, torch's write-only fill, read-only sum, 1:1 copy, and this
library's 1:2 null kernel (the traffic ceiling of the hot path), in GB/s of bytes moved.

  python tools/hbm_probe.py
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_cs_0406049_b200 as sp  # noqa: E402


def timeit(fn, reps=20):
    for _ in range(3):
        fn()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps / 1e3


def main():
    n = 1 << 28
    x = torch.empty(n, dtype=torch.float32, device="cuda").uniform_()
    y = torch.empty(2 * n, dtype=torch.float32, device="cuda")
    s, c = y[:n], y[n:]
    out = {}
    t = timeit(lambda: y.fill_(1.0))
    out["fill_write_only"] = 8 * n / t / 1e9
    t = timeit(lambda: x.sum())
    out["sum_read_only"] = 4 * n / t / 1e9
    t = timeit(lambda: s.copy_(x))
    out["copy_1r1w"] = 8 * n / t / 1e9
    big = torch.empty(2 * n, dtype=torch.float32, device="cuda").uniform_()
    t = timeit(lambda: y.copy_(big))
    out["copy_1r1w_2GiB"] = 16 * n / t / 1e9
    t = timeit(lambda: sp.null_4in8out(x, s, c))
    out["null_1r2w_split"] = 12 * n / t / 1e9
    t = timeit(lambda: sp.null_4in8out(x, interleaved_out=y))
    out["null_1r2w_inter"] = 12 * n / t / 1e9
    t = timeit(lambda: sp.sincos_pairs(x, s, c, variant=0))
    out["sincos_N_split"] = 12 * n / t / 1e9
    # read-only / write-only ceilings in the hot kernel's own access style
    import ctypes
    import subprocess
    so = "/tmp/probe_kernels.so"
    subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-shared",
                           "-Xcompiler", "-fPIC", "-cudart", "static", "-o", so,
                           os.path.join(ROOT, "tools", "probe_kernels.cu")])
    P = ctypes.CDLL(so)
    P.probe_read.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_void_p]
    P.probe_write.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p]
    st = torch.cuda.current_stream().cuda_stream
    t = timeit(lambda: P.probe_read(big.data_ptr(), y.data_ptr(), 2 * n, 0, st))
    out["probe_read_only_256b"] = 8 * n / t / 1e9
    t = timeit(lambda: P.probe_read(big.data_ptr(), y.data_ptr(), 2 * n, 1, st))
    out["probe_read_only_256b_x2"] = 8 * n / t / 1e9
    t = timeit(lambda: P.probe_write(y.data_ptr(), 2 * n, st))
    out["probe_write_only_256b"] = 8 * n / t / 1e9
    print(json.dumps({k: round(v, 1) for k, v in out.items()}))


if __name__ == "__main__":
    main()
