"""One launch each of the phase grid's short-row kernel on short rows (nt = 65, 100 with t one
float off) and of the flat kernel (set_realign(3)) on nt = 65, split, turns, variant N, ~2^30
pairs -- for an ncu capture:
  ncu --set full -k regex:"phase_grid_(short|flat)" python tools/prof_phase_short.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_cs_0406049_b200 as sp  # noqa: E402
from paper_cs_0406049_b200 import ab  # A/B build (tools only)

for nt, toff, mode in ((65, 0, 1), (100, 1, 1), (65, 0, 3)):
    ab.set_realign(mode)
    nf = (1 << 30) // nt
    f = torch.rand(nf, device="cuda") * 512
    t = torch.rand(nt + 8, device="cuda")[toff:toff + nt]
    s = torch.empty(nf * nt, device="cuda")
    c = torch.empty(nf * nt, device="cuda")
    sp.phase_grid(f, t, s, c, units=sp.TURNS)
    torch.cuda.synchronize()
    del s, c
ab.set_realign(1)
print("ok")
