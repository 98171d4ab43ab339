"""One launch each of the traffic patterns around the hot kernel, for an ncu DRAM-activity
capture (GPU box): read-only and write-only probes (tools/probe_kernels.cu), torch's 1:1 copy,
the hot kernel's no-math twin (1 read : 2 writes) and the hot kernel itself.
  ncu --metrics dram__cycles_active.sum,dram__cycles_active_read.sum,dram__cycles_active_write.sum,\
dram__cycles_elapsed.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
      --clock-control none python tools/prof_dram_mix.py"""
import ctypes
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_cs_0406049_b200 as sp  # noqa: E402


def main():
    so = "/tmp/probe_kernels.so"
    subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-shared",
                           "-Xcompiler", "-fPIC", "-cudart", "static", "-o", so,
                           os.path.join(ROOT, "tools", "probe_kernels.cu")])
    P = ctypes.CDLL(so)
    P.probe_read.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_void_p]
    P.probe_write.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p]
    n = 1 << 28
    x = torch.rand(n, device="cuda")
    s, c = torch.empty_like(x), torch.empty_like(x)
    big = torch.rand(2 * n, device="cuda")
    y = torch.empty(2 * n, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    P.probe_read(big.data_ptr(), y.data_ptr(), 2 * n, 0, st)     # 8 GiB... 2n floats read
    P.probe_write(y.data_ptr(), 2 * n, st)
    s.copy_(x)
    sp.null_4in8out(x, s, c)
    sp.sincos_pairs(x, s, c, variant=0)
    torch.cuda.synchronize()
    print("ok")


if __name__ == "__main__":
    main()
