"""The product's phase-grid kernels on the shapes whose traffic mix tools/mix_ceiling_probe.cu
measures without arithmetic (GPU box; run both in one call):

  aligned nt = 2^15 interleaved (write-only stream; f read once per 2^15 pairs),
  staged nt = 5 interleaved (4 B of f per 40 B written), staged nt = 11 split (4 B per 88 B),
  short-row nt = 1001 interleaved,

turns and radians, variant N and A; ~2^30 pairs per launch; median of 5 rounds of 4 launches
(3 warm-up), each case after 3 s idle (burst: the write-heavy grid reaches the board's power cap
within ~0.1 s of sustained load; PHASE_MIX_IDLE=0 for back-to-back cases).  One JSON line per
case: GB/s written and GB/s of traffic (written + f read).
  python tools/phase_mix_compare.py"""
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_cs_0406049_b200 as sp  # noqa: E402


IDLE = float(os.environ.get("PHASE_MIX_IDLE", "3"))


def main():
    dev = torch.device("cuda:0")
    o = torch.empty(2 * (1 << 30) + 64, device=dev)
    s_buf = torch.empty((1 << 30) + 64, device=dev)
    c_buf = torch.empty((1 << 30) + 64, device=dev)
    for nt, inter in ((1 << 15, True), (5, True), (11, False), (1001, True)):
        nf = (1 << 30) // nt
        f = torch.rand(nf, device=dev, generator=torch.Generator(device=dev).manual_seed(5)) * 512
        t = torch.rand(nt, device=dev, generator=torch.Generator(device=dev).manual_seed(6))
        n = nf * nt
        outs = {"interleaved_out": o[:2 * n]} if inter else {"sin_out": s_buf[:n], "cos_out": c_buf[:n]}
        for units, uname in ((sp.TURNS, "turns"), (sp.RADIANS, "radians")):
            for v, vname in ((sp.NORMALIZED, "N"), (sp.RENORMALIZED, "A")):
                def go():
                    sp.phase_grid(f, t, **outs, units=units, variant=v)
                torch.cuda.synchronize()
                time.sleep(IDLE)
                for _ in range(3):
                    go()
                ms = []
                for _ in range(5):
                    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a.record()
                    for _ in range(4):
                        go()
                    b.record()
                    torch.cuda.synchronize()
                    ms.append(a.elapsed_time(b) / 4)
                m = statistics.median(ms)
                wr, rd = 8.0 * n, 4.0 * nf
                print(json.dumps({"nt": nt, "nf": nf, "layout": "interleaved" if inter else "split", "units": uname,
                                  "variant": vname, "ms": round(m, 4), "GBps_written": round(wr / m / 1e6, 1),
                                  "GBps_total": round((wr + rd) / m / 1e6, 1), "ms_min_max": [min(ms), max(ms)]}),
                      flush=True)


if __name__ == "__main__":
    main()
