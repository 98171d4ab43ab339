"""One phase-grid shape, launched twice (for ncu: profile the second launch with
--launch-skip 1 --launch-count 1 -k regex:phase_grid).  Product library, turns, variant N.

  python tools/prof_phase_case.py NT TOFF inter|split"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_cs_0406049_b200 as sp  # noqa: E402

nt, toff, lay = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
nf = (1 << 30) // nt
f = torch.rand(nf, device="cuda") * 512
t = torch.rand(nt + 8, device="cuda")[toff:toff + nt]
n = nf * nt
outs = ({"interleaved_out": torch.empty(2 * n, device="cuda")} if lay == "inter" else
        {"sin_out": torch.empty(n, device="cuda"), "cos_out": torch.empty(n, device="cuda")})
for _ in range(2):
    sp.phase_grid(f, t, units=sp.TURNS, **outs)
torch.cuda.synchronize()
print("ok", nt, toff, lay)
