"""One launch of the hot kernel and of its no-math twin at the C1 size (2^20, split), data
already in L2 (two warm-up launches), for an ncu capture of the latency-bound regime.
  ncu --set full -k regex:sincos_vec_kernel -s 2 -c 3 python tools/prof_small.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import inputs  # noqa: E402
import paper_cs_0406049_b200 as sp  # noqa: E402

n = 1 << 20
th = torch.from_numpy(inputs.generate(1, 0, n)).cuda()
s, c = torch.empty_like(th), torch.empty_like(th)
for _ in range(2):
    sp.sincos_pairs(th, s, c, variant=sp.RENORMALIZED)
sp.sincos_pairs(th, s, c, variant=sp.RENORMALIZED)
sp.sincos_pairs(th, s, c, variant=sp.NORMALIZED)
sp.null_4in8out(th, s, c)
torch.cuda.synchronize()
print("ok")
