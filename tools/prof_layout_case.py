"""One hot-path pointer layout at the C2 size, launched twice (for ncu: --launch-skip 1
--launch-count 1).  Product library, variant N (PROF_VARIANT=1: A).

  python tools/prof_layout_case.py THETA_OFF SIN_OFF COS_OFF    (split)
  python tools/prof_layout_case.py THETA_OFF INTER_OFF          (interleaved)"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_cs_0406049_b200 as sp  # noqa: E402

N = 1 << 28
offs = [int(x) for x in sys.argv[1:]]
tb = torch.rand(N + 16, device="cuda") * 2e4 - 1e4
th = tb[offs[0]:offs[0] + N]
if len(offs) == 3:
    sb, cb = torch.empty(N + 16, device="cuda"), torch.empty(N + 16, device="cuda")
    outs = {"sin_out": sb[offs[1]:offs[1] + N], "cos_out": cb[offs[2]:offs[2] + N]}
else:
    ib = torch.empty(2 * N + 16, device="cuda")
    outs = {"interleaved_out": ib[offs[1]:offs[1] + 2 * N]}
for _ in range(2):
    sp.sincos_pairs(th, **outs, variant=int(os.environ.get("PROF_VARIANT", "0")))
torch.cuda.synchronize()
print("ok", offs)
