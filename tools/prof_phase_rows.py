"""One launch each of the phase grid's row kernel and flat kernel on ragged rows (turns,
variant N, ~2^30 pairs), for an ncu capture:
  ncu --set full -k regex:phase_grid python tools/prof_phase_rows.py
cases: nt = 2^15 - 1 split (rows, flat), nt = 2^15 - 1 interleaved (rows), nt = 4000 with t
at a 5-float offset split (rows), nt = 1001 split (rows), nt = 2^15 + 4 split (rows); an
optional argument skips the first cases."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_cs_0406049_b200 as sp  # noqa: E402
from paper_cs_0406049_b200 import ab  # A/B build (tools only)

CASES = (((1 << 15) - 1, 0, False, 1), ((1 << 15) - 1, 0, False, 3), ((1 << 15) - 1, 0, True, 1),
         (4000, 5, False, 1), (1001, 0, False, 1), ((1 << 15) + 4, 0, False, 1))
for nt, toff, inter, mode in CASES[int(sys.argv[1]):] if len(sys.argv) > 1 else CASES:
    nf = (1 << 30) // nt
    f = torch.rand(nf, device="cuda") * 512
    t = torch.rand(nt + 8, device="cuda")[toff:toff + nt]
    n = nf * nt
    ab.set_realign(mode)
    if inter:
        outs = {"interleaved_out": torch.empty(2 * n, device="cuda")}
    else:
        outs = {"sin_out": torch.empty(n, device="cuda"), "cos_out": torch.empty(n, device="cuda")}
    sp.phase_grid(f, t, units=sp.TURNS, **outs)
    torch.cuda.synchronize()
    del outs
ab.set_realign(1)
print("ok")
