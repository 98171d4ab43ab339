"""GB/s (8 B written per pair) of sincos_phase_grid for row lengths nt with and without the
256-bit row path (nt % 8 == 0 and 32-B aligned t/outputs), split and interleaved (GPU box);
ragged rows through the row kernel (nt >= 128) or the short-row kernel (8 <= nt < 128)
(set_realign(1)) and through the flat kernel (set_realign(3)).
~2^30 pairs per launch.
  python tools/phase_ragged_probe.py"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_cs_0406049_b200 as sp  # noqa: E402
from paper_cs_0406049_b200 import ab  # A/B build (tools only)


MIN_NT = int(os.environ.get("ROWS_MIN_NT", "256"))   # the library's kPhaseRowsMinNt (A/B builds)


def main():
    res = {}
    for nt, toff in ((1 << 15, 0), ((1 << 15) - 1, 0), ((1 << 15) + 4, 0), (1000, 0), (1001, 0), (1001, 3),
                     (9, 0), (33, 0), (65, 0), (100, 1), (127, 0), (131, 0), (200, 2), (255, 0), (300, 0), (500, 1), (4000, 5)):
        nf = (1 << 30) // nt
        f = torch.rand(nf, device="cuda") * 512
        t = torch.rand(nt + 8, device="cuda")[toff:toff + nt]
        n = nf * nt
        for inter, mode in ((False, 1), (True, 1), (False, 3), (True, 3)):
            if mode == 3 and nt % 8 == 0 and toff == 0:
                continue
            ab.set_realign(mode)
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
            kern = "vec" if nt % 8 == 0 and toff == 0 else ("rows" if mode == 1 and nt >= MIN_NT else
                                                             "short" if mode == 1 and nt >= 8 else "flat")
            res[f"nt={nt} toff={toff} {'inter' if inter else 'split'} {kern}"] = round(8 * n / (ms / 1e3) / 1e9, 1)
            del outs
    ab.set_realign(1)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
