"""A/B of libraries on the hot path's pointer layouts (tuning aid; GPU box).

  python tools/ab_layouts.py            # times every tools/ab_layouts/*.so

C2 size (2^28 angles), variant N (AB_VARIANT=1: A): theta / sin / cos / interleaved at the offsets (in floats)
that select each kernel form -- aligned (KB1/KB2), theta off the outputs (KB3b), sin and cos
apart mod 16 B and interleaved pairs only 4-B aligned (KB3c) -- GB/s of 12 B per pair,
median of 5 rounds x 5 launches, the libraries interleaved over rounds.  One JSON line per
library."""
import ctypes
import glob
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
AB = os.path.join(ROOT, "tools", "ab_layouts")
N = 1 << 28
# (name, theta offset, sin offset, cos offset) or (name, theta offset, interleaved offset)
CASES = [("aligned split", 0, 0, 0), ("aligned inter", 0, 0), ("theta+1 split", 1, 0, 0), ("theta+1 inter", 1, 0),
         ("sin+1 cos+2", 0, 1, 2), ("sin+0 cos+3", 0, 0, 3), ("sin+2 cos+5", 0, 2, 5), ("inter+1", 0, 1),
         ("inter+3", 0, 3), ("theta+3 inter+5", 3, 5)]


if os.environ.get("AB_CASES") == "inter":
    CASES = [("aligned split", 0, 0, 0), ("sin+2 cos+5", 0, 2, 5)] + [(f"inter+{a}", 0, a) for a in range(8)]
if os.environ.get("AB_CASES") == "theta":
    # theta at every float offset against aligned split / interleaved outputs, and against
    # outputs that are themselves off (theta and outputs apart in both directions)
    CASES = [(f"theta+{a} split", a, 0, 0) for a in range(8)] + [(f"theta+{a} inter", a, 0) for a in range(8)] + \
            [(f"theta+{a} sin+{b} cos+{b}", a, b, b) for a, b in ((1, 3), (3, 1), (2, 6), (5, 2))] + \
            [(f"theta+{a} inter+{b}", a, b) for a, b in ((1, 4), (3, 5), (2, 7), (6, 1))]
VARIANT = int(os.environ.get("AB_VARIANT", "0"))     # 0 = N, 1 = A


if os.environ.get("AB_CASES") == "all":
    # every split (sin, cos) offset pair 0..7 with theta aligned, and every interleaved offset
    CASES = [(f"sin+{a} cos+{b}", 0, a, b) for a in range(8) for b in range(8)] + \
            [(f"inter+{a}", 0, a) for a in range(8)]


def main():
    import torch
    libs = {}
    for p in sorted(glob.glob(os.path.join(AB, "*.so"))):
        L = ctypes.CDLL(p)
        L.sincos_pairs.restype = ctypes.c_int
        L.sincos_pairs.argtypes = [ctypes.c_void_p] * 4 + [ctypes.c_size_t, ctypes.c_int, ctypes.c_void_p]
        libs[os.path.basename(p)[:-3]] = L
    st = torch.cuda.current_stream().cuda_stream
    tb = torch.rand(N + 16, device="cuda") * 2e4 - 1e4
    sb = torch.empty(N + 16, device="cuda")
    cb = torch.empty(N + 16, device="cuda")
    ib = torch.empty(2 * N + 16, device="cuda")
    res = {k: {} for k in libs}
    for case in CASES:
        name, to = case[0], case[1]
        th = tb.data_ptr() + 4 * to
        if len(case) == 4:
            outs = (sb.data_ptr() + 4 * case[2], cb.data_ptr() + 4 * case[3], None)
        else:
            outs = (None, None, ib.data_ptr() + 4 * case[2])
        samples = {k: [] for k in libs}
        order = list(libs)
        for rnd in range(len(order) * -(-5 // len(order))):   # rotating order (see ab_phase.py)
            for lname in order[rnd % len(order):] + order[:rnd % len(order)]:
                L = libs[lname]
                def go():
                    r = L.sincos_pairs(th, *outs, N, VARIANT, st)
                    assert r == 0, r
                go()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                for _ in range(5):
                    go()
                b.record()
                torch.cuda.synchronize()
                samples[lname].append(a.elapsed_time(b) / 5)
        for lname in libs:
            res[lname][name] = round(12 * N / (statistics.median(samples[lname]) / 1e3) / 1e9, 1)
    for lname in libs:
        print(json.dumps({"lib": lname, "variant": VARIANT, "GBps": res[lname]}))


if __name__ == "__main__":
    main()
