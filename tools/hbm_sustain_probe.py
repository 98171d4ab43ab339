"""GB/s of back-to-back launches from an idle GPU, in groups of 5 launches, with the SM clock,
HBM temperature, board power and throttle reasons after each group (GPU box):
  python tools/hbm_sustain_probe.py > profiles/hbm_sustain_r01.json
Forms: the hot path (C2: 2^28 angles, split, variant N; 12 B/pair, 1:2 read/write), its
no-math twin, the phase grid (2^30 pairs, write-only 8 B/pair) and a torch copy (1 GiB).
Each form starts after 3 s idle.  Shows how throughput depends on how long the memory has been
under load (the reason the bench reports both its time-averaged value and a burst figure)."""
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


def state(h):
    try:
        mt = pynvml.nvmlDeviceGetFieldValues(h, [pynvml.NVML_FI_DEV_MEMORY_TEMP])[0]
        mem_t = mt.value.uiVal if mt.nvmlReturn == 0 else None
    except pynvml.NVMLError:
        mem_t = None
    return {"sm_mhz": pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
            "mem_temp_c": mem_t,
            "gpu_temp_c": pynvml.nvmlDeviceGetTemperature(h, 0),
            "power_w": pynvml.nvmlDeviceGetPowerUsage(h) // 1000,
            "reasons": hex(pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(h))}


def series(h, fn, nbytes, groups=80):
    out = []
    t0 = time.time()
    for _ in range(groups):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(5):
            fn()
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / 5
        out.append({"t_s": round(time.time() - t0, 3), "gbs": round(nbytes / (ms / 1e3) / 1e9, 1), **state(h)})
    return out


def main():
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
    n = 1 << 28
    th = torch.from_numpy(inputs.generate(2, 0, n)).cuda()
    s, c = torch.empty(n, device="cuda"), torch.empty(n, device="cuda")
    nt = nf = 1 << 15
    f, t = torch.rand(nf, device="cuda") * 512, torch.rand(nt, device="cuda")
    ps, pc = torch.empty(nf * nt, device="cuda"), torch.empty(nf * nt, device="cuda")
    x = torch.empty(1 << 28, device="cuda")
    y = torch.empty(1 << 28, device="cuda")
    forms = {
        "hot_path_c2_split_N": (lambda: sp.sincos_pairs(th, s, c, variant=0), 12 * n),
        "null_twin_c2_split": (lambda: sp.null_4in8out(th, s, c), 12 * n),
        "phase_grid_2p30_split": (lambda: sp.phase_grid(f, t, ps, pc, units=sp.TURNS), 8 * nf * nt),
        "torch_copy_1GiB": (lambda: y.copy_(x), 8 * (1 << 28)),
    }
    res = {"note": "groups of 5 back-to-back launches after 3 s idle; gbs = bytes moved per launch / mean launch time"}
    for name, (fn, nbytes) in forms.items():
        fn()
        torch.cuda.synchronize()
        time.sleep(3)
        res[name] = series(h, fn, nbytes)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
