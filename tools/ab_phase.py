"""A/B of build-time switches of libsincos_pairs.so on sincos_phase_grid (tuning aid).

  python tools/ab_phase.py build NAME -DMACRO=V ...   # here (CPU): builds tools/ab_phase/NAME.so
  python tools/ab_phase.py run                        # GPU box: times every tools/ab_phase/*.so
  python tools/ab_phase.py sustain                    # GPU box: 0.5-1 s of load per library from idle

Cases: ragged row lengths (and t offsets) at ~2^30 pairs per launch, split and interleaved,
turns, variant N (AB_VARIANT=1: A; AB_UNITS=0: radians); GB/s of the 8 B written per pair, median
over rounds of 5 launches (at least 5 rounds, a multiple of the library count), the libraries
interleaved over rounds in a rotating order (the first after an AB_BURST idle gap runs cooler: two
identical libraries read 5-8% apart on interleaved nt = 3 without the rotation).  One JSON line
per library."""
import ctypes
import glob
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
AB = os.path.join(ROOT, "tools", "ab_phase")
CASES = [(32767, 0), (32772, 0), (1001, 0), (1001, 3), (4000, 5), (255, 0), (300, 0), (500, 1), (131, 0),
         (65, 0), (100, 1), (200, 2)]
if os.environ.get("AB_CASES") == "short":
    CASES = [(1, 0), (3, 0), (5, 1), (7, 2), (9, 0), (17, 3), (33, 0), (65, 0), (100, 1), (127, 0)]
if os.environ.get("AB_CASES") == "mid":
    CASES = [(131, 0), (200, 2), (255, 0), (300, 0), (500, 1), (1001, 0), (1001, 3), (2000, 0), (4000, 5)]
if os.environ.get("AB_CASES") == "r02":
    CASES = [(1001, 0), (1001, 3), (1, 0), (2, 0), (3, 0), (5, 1), (7, 2), (9, 0), (65, 0), (500, 1), (1000, 0)]
if os.environ.get("AB_CASES") == "tiny":
    CASES = [(1, 0), (2, 0), (3, 0), (4, 0), (5, 1), (6, 0), (7, 2), (9, 0)]
if os.environ.get("AB_CASES") == "rows":
    CASES = [(32767, 0), (32772, 0), (16385, 1), (8191, 3), (4000, 5), (2049, 0), (1025, 2)]
if os.environ.get("AB_CASES") == "small":
    CASES = [(8, 0), (10, 0), (12, 0), (16, 0), (20, 0), (24, 0), (32, 0), (48, 0), (63, 0)]
if os.environ.get("AB_CASES") == "mid8":
    CASES = [(7, 2), (8, 0), (9, 0), (10, 0), (11, 3), (12, 0), (13, 0), (14, 0), (15, 1)]
if os.environ.get("AB_CASES") == "mid16":
    CASES = [(14, 0), (16, 0), (17, 1), (20, 0), (23, 2), (24, 0), (28, 0), (30, 3), (31, 0), (33, 0)]
if os.environ.get("AB_CASES") == "vec8":
    CASES = [(16, 0), (32, 0), (64, 0), (96, 0), (128, 0), (200, 0), (248, 0), (256, 0)]
if os.environ.get("AB_CASES") == "aligned":
    CASES = [(32768, 0), (8192, 0), (4096, 0), (2048, 0), (1000, 0), (512, 0), (256, 0), (136, 0), (64, 0), (16, 0)]


VARIANT = int(os.environ.get("AB_VARIANT", "0"))     # 0 = N, 1 = A
UNITS = int(os.environ.get("AB_UNITS", "1"))         # 1 = turns, 0 = radians
BURST = float(os.environ.get("AB_BURST", "0"))       # > 0: seconds idle before every case (burst figures)


def build(name, flags):
    from paper_cs_0406049_b200 import _build
    os.makedirs(AB, exist_ok=True)
    out = os.path.join(AB, name + ".so")
    _build.build(extra_flags=flags, out=out)
    print(out)


def run():
    import torch
    libs = {}
    for p in sorted(glob.glob(os.path.join(AB, "*.so"))):
        L = ctypes.CDLL(p)
        L.sincos_phase_grid.restype = ctypes.c_int
        L.sincos_phase_grid.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p, ctypes.c_size_t,
                                        ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int,
                                        ctypes.c_int, ctypes.c_void_p]
        libs[os.path.basename(p)[:-3]] = L
    st = torch.cuda.current_stream().cuda_stream
    s = torch.empty(1 << 30, device="cuda")
    c = torch.empty(1 << 30, device="cuda")
    io = torch.empty(1 << 31, device="cuda")
    res = {k: {} for k in libs}
    for nt, toff in CASES:
        nf = (1 << 30) // nt
        f = torch.rand(nf, device="cuda") * 512
        t = torch.rand(nt + 8, device="cuda")[toff:toff + nt]
        for inter in (False, True):
            key = f"nt={nt} toff={toff} {'inter' if inter else 'split'}"
            outs = (0, 0, io.data_ptr()) if inter else (s.data_ptr(), c.data_ptr(), 0)
            samples = {k: [] for k in libs}
            if BURST:
                import time
                torch.cuda.synchronize()
                time.sleep(BURST)                  # let the board leave its power cap
            names = list(libs)
            rounds = len(names) * -(-5 // len(names))   # >= 5, a multiple of the library count
            for rnd in range(rounds):
                # the first library after the idle gap runs cooler: rotate the order every round
                for name in names[rnd % len(names):] + names[:rnd % len(names)]:
                    L = libs[name]
                    def go():
                        r = L.sincos_phase_grid(f.data_ptr(), nf, t.data_ptr(), nt, *outs, UNITS, VARIANT, st)
                        assert r == 0, r
                    go()
                    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a.record()
                    for _ in range(5):
                        go()
                    b.record()
                    torch.cuda.synchronize()
                    samples[name].append(a.elapsed_time(b) / 5)
            for name in libs:
                res[name][key] = round(8 * nf * nt / (statistics.median(samples[name]) / 1e3) / 1e9, 1)
    for name in libs:
        print(json.dumps({"lib": name, "variant": VARIANT, "units": UNITS, "GBps": res[name]}))


def sustain():
    """Per library, twice (alternating), after 3 s idle: 100 groups of 5 launches of the aligned
    C4 shape (2^15 x 2^15, split, turns, variant N): GB/s of the first 5 groups and of the last
    20, the SM clock at the end, and board energy per launch (NVML total-energy counter)."""
    import time

    import pynvml
    import torch
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
    libs = {}
    for p in sorted(glob.glob(os.path.join(AB, "*.so"))):
        L = ctypes.CDLL(p)
        L.sincos_phase_grid.restype = ctypes.c_int
        L.sincos_phase_grid.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p, ctypes.c_size_t,
                                        ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int,
                                        ctypes.c_int, ctypes.c_void_p]
        libs[os.path.basename(p)[:-3]] = L
    st = torch.cuda.current_stream().cuda_stream
    nf = nt = 1 << 15
    f = torch.rand(nf, device="cuda") * 512
    t = torch.rand(nt, device="cuda")
    s = torch.empty(nf * nt, device="cuda")
    c = torch.empty(nf * nt, device="cuda")
    nbytes = 8 * nf * nt
    inter = os.environ.get("SUSTAIN_INTER") == "1"      # interleaved output (s viewed as 2 x n/2... below)
    io = torch.empty(2 * nf * nt, device="cuda") if inter else None
    outs = (0, 0, io.data_ptr()) if inter else (s.data_ptr(), c.data_ptr(), 0)
    out = {k: [] for k in libs}
    for rep in range(2):
        for name, L in libs.items():
            L.sincos_phase_grid(f.data_ptr(), nf, t.data_ptr(), nt, *outs, 1, 0, st)
            torch.cuda.synchronize()
            time.sleep(3)
            e0 = pynvml.nvmlDeviceGetTotalEnergyConsumption(h)
            gbs = []
            for _ in range(100):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                for _ in range(5):
                    L.sincos_phase_grid(f.data_ptr(), nf, t.data_ptr(), nt, *outs, 1, 0, st)
                b.record()
                torch.cuda.synchronize()
                gbs.append(nbytes / (a.elapsed_time(b) / 5 / 1e3) / 1e9)
            mj = pynvml.nvmlDeviceGetTotalEnergyConsumption(h) - e0
            out[name].append({"first5_gbs": round(statistics.mean(gbs[:5]), 1),
                              "last20_gbs": round(statistics.mean(gbs[-20:]), 1),
                              "sm_mhz_end": pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                              "reasons_end": hex(pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(h)),
                              "mJ_per_launch": round(mj / 500, 2)})
    for name in libs:
        print(json.dumps({"lib": name, "sustain": out[name]}))


if __name__ == "__main__":
    if sys.argv[1] == "build":
        build(sys.argv[2], sys.argv[3:])
    elif sys.argv[1] == "sustain":
        sustain()
    else:
        run()
