"""Small invocations of every kernel family for compute-sanitizer (GPU box):
  compute-sanitizer --tool memcheck python tools/sanitize_smoke.py
Covers the vector, 128-bit, re-aligning and one-per-thread forms of the hot path (both
layouts, both variants, ragged lengths), 16-bit outputs, general methods, the phase grid (row
and flat kernels), the fused sum, the host-buffer path and the stats kernel."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_cs_0406049_b200 as sp  # noqa: E402


def main():
    base = torch.rand(5000, device="cuda") * 200 - 100
    for n in (1, 7, 9, 1003):
        for ot in range(8):
            for oo in (0, 1, 3, 4):
                t = base[ot:ot + n]
                s = torch.empty(n + 8, device="cuda")[oo:oo + n]
                c = torch.empty(n + 8, device="cuda")[oo:oo + n]
                io = torch.empty(2 * n + 8, device="cuda")[oo:oo + 2 * n]
                for v in (0, 1):
                    sp.sincos_pairs(t, s, c, variant=v)
                    sp.sincos_pairs(t, interleaved_out=io, variant=v)
                s16 = torch.empty(n + 8, dtype=torch.float16, device="cuda")[oo:oo + n]
                c16 = torch.empty(n + 8, dtype=torch.float16, device="cuda")[oo:oo + n]
                sp.sincos_pairs_dtype(t, s16, c16)
                m = sp.make_method(*sp.PAPER_METHODS[1])
                sp.sincos_pairs_method(t, m, s, c)
                sp.sincos_pairs_method(t, m, interleaved_out=io)
    f = torch.rand(37, device="cuda") * 50
    for nt in (1, 8, 13, 256, 1001):
        tt = torch.rand(nt + 1, device="cuda")[1:]
        o = torch.empty(2 * 37 * nt, device="cuda")
        sp.phase_grid(f, tt, interleaved_out=o, units=sp.TURNS)
        a = torch.randn(nt, dtype=torch.complex64, device="cuda")
        sp.nudft(f, tt, a, units=sp.TURNS)
    th = torch.rand(100_003) * 10
    sh = torch.empty_like(th).pin_memory()
    ch = torch.empty_like(th).pin_memory()
    ws = torch.empty(sp.host_workspace_min_bytes(), dtype=torch.uint8, device="cuda")
    sp.sincos_pairs_host(th.pin_memory(), sh, ch, workspace=ws)
    td = th.cuda()
    sd, cd = sp.sincos(td)
    sp.error_stats(td, sd, cd)
    torch.cuda.synchronize()
    print("sanitize smoke ok")


if __name__ == "__main__":
    main()
