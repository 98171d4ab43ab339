"""Board energy per launch (NVML total-energy counter, >= 2 s of back-to-back launches) of the
hot kernel (variants N and A), its no-math twin and CUDA's sincosf / __sincosf in the same
kernel shape, on the C2 batch (GPU box): how much of the ~1 kW goes to the arithmetic.
  python tools/energy_probe.py"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import pynvml  # noqa: E402
import torch  # noqa: E402

import inputs  # noqa: E402
import paper_cs_0406049_b200 as sp  # noqa: E402


def main():
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(int(os.environ.get("CUDA_VISIBLE_DEVICES", "0").split(",")[0] or 0))
    n = 1 << 28
    th = torch.from_numpy(inputs.generate(2, 0, n)).cuda()
    s, c = torch.empty_like(th), torch.empty_like(th)
    cases = {"method_N": lambda: sp.sincos_pairs(th, s, c, variant=0),
             "method_A": lambda: sp.sincos_pairs(th, s, c, variant=1),
             "no_math_ceiling": lambda: sp.null_4in8out(th, s, c),
             "cuda_sincosf": lambda: sp.compare_cuda(th, s, c, which=3),
             "cuda___sincosf": lambda: sp.compare_cuda(th, s, c, which=4)}
    out = {}
    for name, fn in cases.items():
        for _ in range(20):
            fn()
        torch.cuda.synchronize()
        k = 4200
        e0, t0 = pynvml.nvmlDeviceGetTotalEnergyConsumption(h), time.perf_counter()
        for _ in range(k):
            fn()
        torch.cuda.synchronize()
        e1, t1 = pynvml.nvmlDeviceGetTotalEnergyConsumption(h), time.perf_counter()
        j = (e1 - e0) / 1e3
        out[name] = {"ms_per_launch": 1e3 * (t1 - t0) / k, "mean_power_w": j / (t1 - t0),
                     "mJ_per_launch": 1e3 * j / k, "pairs_per_joule": n * k / j,
                     "sm_mhz_end": pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
