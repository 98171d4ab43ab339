"""GB/s (8 B written per pair) of sincos_phase_grid for row lengths nt with and without the
256-bit path (nt % 8 == 0 and 32-B aligned t/outputs), split and interleaved (GPU box).
  python tools/phase_ragged_probe.py"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_cs_0406049_b200 as sp  # noqa: E402


def main():
    res = {}
    nf = 1 << 15
    for nt in (1 << 15, (1 << 15) - 1, (1 << 15) + 4, 1000, 1001):
        f = torch.rand(nf, device="cuda") * 512
        t = torch.rand(nt, device="cuda")
        n = nf * nt
        for inter in (False, True):
            if inter:
                outs = {"interleaved_out": torch.empty(2 * n, device="cuda")}
            else:
                outs = {"sin_out": torch.empty(n, device="cuda"), "cos_out": torch.empty(n, device="cuda")}
            for _ in range(2):
                sp.phase_grid(f, t, units=sp.TURNS, **outs)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(5):
                sp.phase_grid(f, t, units=sp.TURNS, **outs)
            b.record()
            torch.cuda.synchronize()
            ms = a.elapsed_time(b) / 5
            res[f"nt={nt} {'inter' if inter else 'split'}"] = round(8 * n / (ms / 1e3) / 1e9, 1)
            del outs
    print(json.dumps(res))


if __name__ == "__main__":
    main()
