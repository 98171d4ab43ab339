"""The fused sum (C4 shape, packed, N, turns and radians) run back to back for ~3 s: per-launch
time in the first and the last 10% of the run, SM clock and board power sampled by NVML during
it (GPU box) -- does the FP32-pipe roofline's 1.965 GHz hold under sustained load?
  python tools/sustained_nudft.py"""
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import pynvml  # noqa: E402
import torch  # noqa: E402

import paper_cs_0406049_b200 as sp  # noqa: E402
from bench import c4_axes  # noqa: E402


def main():
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(0)
    nt = 1 << 15
    rng = np.random.default_rng(7)
    a = torch.from_numpy((rng.normal(size=nt) + 1j * rng.normal(size=nt)).astype(np.complex64)).cuda()
    out = {}
    for units, uname in ((sp.TURNS, "turns"), (sp.RADIANS, "radians")):
        f, t = c4_axes(units == sp.TURNS)
        fd, td = torch.from_numpy(f).cuda(), torch.from_numpy(t).cuda()
        o = torch.empty(nt, dtype=torch.complex64, device="cuda")
        ws = torch.empty(sp.lib().sincos_nudft_workspace_bytes(nt, nt), dtype=torch.uint8, device="cuda")
        k = 3000
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(k + 1)]
        clocks, power, stop = [], [], threading.Event()

        def sample():
            while not stop.is_set():
                clocks.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
                power.append(pynvml.nvmlDeviceGetPowerUsage(h) / 1e3)
                time.sleep(0.01)
        th = threading.Thread(target=sample, daemon=True)
        th.start()
        ev[0].record()
        for i in range(k):
            sp.nudft(fd, td, a, out=o, units=units, workspace=ws)
            ev[i + 1].record()
        torch.cuda.synchronize()
        stop.set()
        th.join()
        ms = [ev[i].elapsed_time(ev[i + 1]) for i in range(k)]
        first, last = statistics.median(ms[: k // 10]), statistics.median(ms[-k // 10:])
        out[uname] = {"launches": k, "seconds": sum(ms) / 1e3,
                      "first_10pct_T_terms_per_s": nt * nt / (first / 1e3) / 1e12,
                      "last_10pct_T_terms_per_s": nt * nt / (last / 1e3) / 1e12,
                      "sm_mhz_median": statistics.median(clocks), "sm_mhz_min": min(clocks),
                      "power_w_median": statistics.median(power), "power_w_max": max(power)}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
