"""One launch of each hot-path kernel form on the C2 batch (2^28 angles), for an ncu capture:
variant N and A at unroll U = 1, 2, 4 (split), N and A interleaved (U = 1), the traffic-ceiling
kernel (no math).
  ncu --set full --clock-control none -k regex:sincos_vec_kernel -c 9 python tools/prof_hot.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import inputs  # noqa: E402
import paper_cs_0406049_b200 as sp  # noqa: E402
from paper_cs_0406049_b200 import ab  # A/B build (tools only)


def main():
    n = 1 << 28
    th = torch.from_numpy(inputs.generate(2, 0, n)).cuda()
    s = torch.empty(n, device="cuda")
    c = torch.empty(n, device="cuda")
    io = torch.empty(2 * n, device="cuda")
    for u in (1, 2, 4):
        ab.set_launch_config(unroll=u)
        for v in (sp.NORMALIZED, sp.RENORMALIZED):
            sp.sincos_pairs(th, s, c, variant=v)
    ab.set_launch_config()
    for v in (sp.NORMALIZED, sp.RENORMALIZED):
        sp.sincos_pairs(th, interleaved_out=io, variant=v)
    sp.null_4in8out(th, s, c)
    torch.cuda.synchronize()
    print("ok")


if __name__ == "__main__":
    main()
