"""One launch of the hot kernel (variant N) at each BASELINE config's size and layout, after two
warm-up launches, for an ncu DRAM-traffic capture (GPU box):
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
      -k regex:sincos_vec_kernel --csv python tools/prof_configs.py
C1 split 2^20, C2 split 2^28, C3 interleaved 2^24, C4 interleaved 2^30, C5 split 2^32."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_cs_0406049_b200 as sp  # noqa: E402

for lg, inter in ((20, False), (28, False), (24, True), (30, True), (32, False)):
    n = 1 << lg
    th = torch.rand(n, device="cuda") * 200 - 100
    if inter:
        o = {"interleaved_out": torch.empty(2 * n, device="cuda")}
    else:
        o = {"sin_out": torch.empty(n, device="cuda"), "cos_out": torch.empty(n, device="cuda")}
    for _ in range(3):
        sp.sincos_pairs(th, **o)
    torch.cuda.synchronize()
    del th, o
    torch.cuda.empty_cache()
print("ok")
