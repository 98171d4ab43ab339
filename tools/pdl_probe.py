"""A/B of programmatic dependent launch (the A/B build's pdl knob) on back-to-back steps (variant N then
A, split) at 2^20 .. 2^28 elements: plain stream launches and a CUDA graph of 20 steps
(GPU box).  python tools/pdl_probe.py"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_cs_0406049_b200 as sp  # noqa: E402
from paper_cs_0406049_b200 import ab  # A/B build (tools only)


def time_steps(th, s, c, graph, steps=20, reps=5):
    def step(st=None):
        sp.sincos_pairs(th, s, c, variant=0, stream=st)
        sp.sincos_pairs(th, s, c, variant=1, stream=st)
    for _ in range(3):
        step()
    if graph:
        cap = torch.cuda.Stream()
        cap.wait_stream(torch.cuda.current_stream())
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=cap):
            for _ in range(steps):
                step(cap)
        torch.cuda.current_stream().wait_stream(cap)
        g.replay()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        if graph:
            g.replay()
        else:
            for _ in range(steps):
                step()
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b) / steps)
    return best * 1e3   # us per step


def main():
    res = {}
    for lg in (20, 22, 24, 28):
        n = 1 << lg
        th = torch.rand(n, device="cuda") * 2e4 - 1e4
        s, c = torch.empty_like(th), torch.empty_like(th)
        for graph in (False, True):
            for pdl in (False, True, False, True):
                ab.set_pdl(pdl)
                us = time_steps(th, s, c, graph)
                key = f"2^{lg} {'graph' if graph else 'stream'} pdl={int(pdl)}"
                res[key] = min(res.get(key, 1e18), round(us, 2))
    ab.set_pdl(True)
    print(json.dumps({"us_per_step_N_then_A": res}))


if __name__ == "__main__":
    main()
