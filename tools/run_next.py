"""Run each NEXT-row kernel once at the C4 shape (for ncu captures): the phase grid
(sincos_phase_grid, radians, interleaved) and the fused sum (sincos_nudft, radians), variant N
then A.  python tools/run_next.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_cs_0406049_b200 as sp  # noqa: E402
from bench import c4_axes  # noqa: E402


def main():
    f, t = c4_axes(turns=False)
    fd, td = torch.from_numpy(f).cuda(), torch.from_numpy(t).cuda()
    o = torch.empty(2 << 30, device="cuda")
    rng = np.random.default_rng(7)
    a = torch.from_numpy((rng.normal(size=t.size) + 1j * rng.normal(size=t.size)).astype(np.complex64)).cuda()
    for v in (sp.NORMALIZED, sp.RENORMALIZED):
        sp.phase_grid(fd, td, interleaved_out=o, units=sp.RADIANS, variant=v)
        out = sp.nudft(fd, td, a, units=sp.RADIANS, variant=v)
    torch.cuda.synchronize()
    print("ok", out[:2].cpu().numpy())


if __name__ == "__main__":
    main()
