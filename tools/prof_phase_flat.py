"""One launch each of the phase grid's vector kernel (nt = 2^15) and flat kernel (nt = 2^15 - 1),
split, turns, variant N, for an ncu capture.
  ncu --set full -k regex:phase_grid -c 2 python tools/prof_phase_flat.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_cs_0406049_b200 as sp  # noqa: E402

nf = 1 << 15
for nt in (1 << 15, (1 << 15) - 1):
    f = torch.rand(nf, device="cuda") * 512
    t = torch.rand(nt, device="cuda")
    s = torch.empty(nf * nt, device="cuda")
    c = torch.empty(nf * nt, device="cuda")
    sp.phase_grid(f, t, s, c, units=sp.TURNS)
    torch.cuda.synchronize()
    del s, c
print("ok")
