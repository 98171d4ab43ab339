"""One launch of each fused-sum kernel form at the C4 shape, for an ncu capture:
packed / scalar x radians / turns (variant N), then packed method (1; 3, 2) in turns.
  ncu --set full --clock-control none -k regex:nudft_partial -c 5 python tools/prof_nudft.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_cs_0406049_b200 as sp  # noqa: E402
from paper_cs_0406049_b200 import ab  # A/B build (tools only)
from bench import c4_axes, fit_method  # noqa: E402


def main():
    nt = 1 << 15
    rng = np.random.default_rng(7)
    a = torch.from_numpy((rng.normal(size=nt) + 1j * rng.normal(size=nt)).astype(np.complex64)).cuda()
    for packed, units, kw in ((1, sp.RADIANS, {"variant": 0}), (1, sp.TURNS, {"variant": 0}),
                              (0, sp.RADIANS, {"variant": 0}), (0, sp.TURNS, {"variant": 0}),
                              (1, sp.TURNS, {"method": fit_method(1, 3, 2)})):
        ab.set_nudft_packed(bool(packed))
        f, t = c4_axes(units == sp.TURNS)
        sp.nudft(torch.from_numpy(f).cuda(), torch.from_numpy(t).cuda(), a, units=units, **kw)
    torch.cuda.synchronize()
    print("ok")


if __name__ == "__main__":
    main()
