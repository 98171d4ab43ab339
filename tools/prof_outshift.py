"""One launch each of the output-realigning kernel (KB3c), split with sin / cos apart and
interleaved with 4-B pairs, plus the aligned kernel, at the C2 size -- for an ncu capture.
  ncu --set full -k regex:"outshift|sincos_vec_kernel" -c 3 python tools/prof_outshift.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_cs_0406049_b200 as sp  # noqa: E402

n = 1 << 28
th = torch.rand(n, device="cuda") * 2e4 - 1e4
sb, cb = torch.empty(n + 8, device="cuda"), torch.empty(n + 8, device="cuda")
ib = torch.empty(2 * n + 8, device="cuda")
sp.sincos_pairs(th, sb[:n], cb[:n])
sp.sincos_pairs(th, sb[1:1 + n], cb[2:2 + n])
sp.sincos_pairs(th, interleaved_out=ib[1:1 + 2 * n])
torch.cuda.synchronize()
print("ok")
