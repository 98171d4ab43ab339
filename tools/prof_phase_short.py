"""One launch each of the phase grid's flat kernel on short rows (nt = 65, 100 with t one float
off), split, turns, variant N, ~2^30 pairs -- for an ncu capture:
  ncu --set full -k regex:phase_grid_flat python tools/prof_phase_short.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_cs_0406049_b200 as sp  # noqa: E402

for nt, toff in ((65, 0), (100, 1)):
    nf = (1 << 30) // nt
    f = torch.rand(nf, device="cuda") * 512
    t = torch.rand(nt + 8, device="cuda")[toff:toff + nt]
    s = torch.empty(nf * nt, device="cuda")
    c = torch.empty(nf * nt, device="cuda")
    sp.phase_grid(f, t, s, c, units=sp.TURNS)
    torch.cuda.synchronize()
    del s, c
print("ok")
