"""A/B of libraries on the fused sum (GPU box): every tools/ab_nudft/*.so on the C4 shape
(2^15 x 2^15 terms, bench.py's axes), variants N and A, radians and turns; T terms/s, median
of 5 rounds x 5 launches with the libraries' order rotating every round; outputs compared
between libraries (max |difference|, 0 when the arithmetic is unchanged).  One JSON line.
  python tools/ab_nudft.py"""
import ctypes
import glob
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from bench import c4_axes  # noqa: E402

AB = os.path.join(ROOT, "tools", "ab_nudft")


def main():
    libs = {}
    for p in sorted(glob.glob(os.path.join(AB, "*.so"))):
        L = ctypes.CDLL(p)
        L.sincos_nudft.restype = ctypes.c_int
        L.sincos_nudft.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t,
                                   ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_size_t,
                                   ctypes.c_void_p]
        L.sincos_nudft_workspace_bytes.restype = ctypes.c_size_t
        L.sincos_nudft_workspace_bytes.argtypes = [ctypes.c_size_t, ctypes.c_size_t]
        libs[os.path.basename(p)[:-3]] = L
    nf = nt = 1 << 15
    rng = np.random.default_rng(7)
    a = torch.from_numpy((rng.normal(size=nt) + 1j * rng.normal(size=nt)).astype(np.complex64)).cuda()
    ar = torch.view_as_real(a).contiguous()
    st = torch.cuda.current_stream().cuda_stream
    res = {}
    for units, uname in ((1, "turns"), (0, "radians")):
        f, t = c4_axes(units == 1)
        fd, td = torch.from_numpy(f).cuda(), torch.from_numpy(t).cuda()
        for v, vname in ((0, "N"), (1, "A")):
            outs, samples = {}, {k: [] for k in libs}
            for k, L in libs.items():
                ws = torch.empty(int(L.sincos_nudft_workspace_bytes(nf, nt)), dtype=torch.uint8, device="cuda")
                outs[k] = (torch.empty(nf, dtype=torch.complex64, device="cuda"), ws)
            order = list(libs)
            for rnd in range(len(order) * -(-5 // len(order))):
                for k in order[rnd % len(order):] + order[:rnd % len(order)]:
                    L, (o, ws) = libs[k], outs[k]

                    def go():
                        r = L.sincos_nudft(fd.data_ptr(), nf, td.data_ptr(), ar.data_ptr(), nt,
                                           torch.view_as_real(o).data_ptr(), units, v, ws.data_ptr(), ws.numel(), st)
                        assert r == 0, r
                    go()
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                    for _ in range(5):
                        go()
                    e1.record()
                    torch.cuda.synchronize()
                    samples[k].append(e0.elapsed_time(e1) / 5)
            ref = outs[order[0]][0]
            for k in libs:
                ms = statistics.median(samples[k])
                res.setdefault(k, {})[f"{uname}_{vname}"] = {
                    "ms": round(ms, 4), "T_terms_per_s": round(nf * nt / (ms / 1e3) / 1e12, 4),
                    "max_abs_diff_vs_first": float((outs[k][0] - ref).abs().max())}
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
