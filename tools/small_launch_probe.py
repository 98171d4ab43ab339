"""Per-launch time of the hot kernel at L2-resident sizes (2^16 .. 2^24) for launch
configurations, each timed as a CUDA graph of 50 back-to-back launches (GPU box).
  python tools/small_launch_probe.py"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_cs_0406049_b200 as sp  # noqa: E402
from paper_cs_0406049_b200 import ab  # A/B build (tools only)

CFGS = [(128, 0, 8, 1, 0), (256, 0, 8, 1, 0), (512, 0, 8, 1, 0), (128, 0, 4, 1, 0), (256, 0, 4, 1, 0),
        (128, 0, 8, 2, 0), (256, 2, 8, 1, 0), (512, 1, 8, 1, 0)]


def main():
    res = {}
    for lg in (16, 18, 20, 22, 24):
        n = 1 << lg
        th = torch.rand(n, device="cuda") * 100
        s, c = torch.empty_like(th), torch.empty_like(th)
        for cfg in CFGS:
            ab.set_launch_config(*cfg)
            for _ in range(3):
                sp.sincos_pairs(th, s, c)
            cap = torch.cuda.Stream()
            cap.wait_stream(torch.cuda.current_stream())
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=cap):
                for _ in range(50):
                    sp.sincos_pairs(th, s, c, stream=cap)
            torch.cuda.current_stream().wait_stream(cap)
            g.replay()
            torch.cuda.synchronize()
            best = 1e9
            for _ in range(5):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                g.replay()
                b.record()
                torch.cuda.synchronize()
                best = min(best, a.elapsed_time(b) / 50 * 1e3)
            res.setdefault(f"2^{lg}", {})[",".join(map(str, cfg))] = round(best, 2)
    ab.set_launch_config()
    print(json.dumps({"us_per_launch": res}))


if __name__ == "__main__":
    main()
