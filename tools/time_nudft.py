"""Time the fused sum (sincos_nudft) at the C4 shape for a quick A/B of kernel changes.
python tools/time_nudft.py"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_cs_0406049_b200 as sp  # noqa: E402
from paper_cs_0406049_b200 import ab  # A/B build (tools only)
from bench import c4_axes, fit_method  # noqa: E402


def main():
    nf = nt = 1 << 15
    rng = np.random.default_rng(7)
    a = torch.from_numpy((rng.normal(size=nt) + 1j * rng.normal(size=nt)).astype(np.complex64)).cuda()
    out = {}
    packed = os.environ.get("NUDFT_PACKED")
    if packed is not None:
        ab.set_nudft_packed(packed == "1")
    for units in (sp.RADIANS, sp.TURNS):
        f, t = c4_axes(units == sp.TURNS)
        fd, td = torch.from_numpy(f).cuda(), torch.from_numpy(t).cuda()
        for name, kw in (("N", {"variant": 0}), ("A", {"variant": 1}), ("m132", {"method": fit_method(1, 3, 2)}),
                         ("m332_general", {"method": fit_method(3, 3, 2)}),
                         ("m254_general", {"method": fit_method(2, 5, 4)})):
            sp.nudft(fd, td, a, units=units, **kw)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(10):
                sp.nudft(fd, td, a, units=units, **kw)
            e1.record()
            torch.cuda.synchronize()
            out[f"{'rt'[units]}_{name}"] = round(nf * nt / (e0.elapsed_time(e1) / 10 / 1e3) / 1e12, 4)
    print(json.dumps({"packed": packed, "T_terms_per_s": out}))


if __name__ == "__main__":
    main()
