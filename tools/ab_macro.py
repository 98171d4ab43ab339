"""A/B of build-time switches of libsincos_pairs.so on the hot path (tuning aid).

  python tools/ab_macro.py build NAME -DMACRO=V ...   # here (CPU): builds tools/ab/NAME.so
  python tools/ab_macro.py run                        # GPU box: times every tools/ab/*.so
  python tools/ab_macro.py energy                     # GPU box: 2 s of C2 launches per library, J/launch
  python tools/ab_macro.py method                     # GPU box: sincos_pairs_method (paper tables) per library

Times variants N and A, split and interleaved, on the C2 batch (2^28 angles, 12 B/pair),
the libraries interleaved over rounds (median of 5 rounds x 10 launches).  One JSON line
per library.  The default build (no switches) should be built as a control."""
import ctypes
import glob
import json
import os
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
AB = os.path.join(ROOT, "tools", "ab")


def build(name, flags):
    from paper_cs_0406049_b200 import _build
    os.makedirs(AB, exist_ok=True)
    out = os.path.join(AB, name + ".so")
    _build.build(extra_flags=flags, out=out)
    print(out)


def run():
    import torch

    import inputs
    n = int(os.environ.get("AB_N", 1 << 28))
    graph = 12 * n < (256 << 20)          # launch-bound sizes: time a graph of 20 launches
    th = torch.from_numpy(inputs.generate(2, 0, n)).cuda()
    s = torch.empty(n, device="cuda")
    c = torch.empty(n, device="cuda")
    io = torch.empty(2 * n, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    libs = {}
    for p in sorted(glob.glob(os.path.join(AB, "*.so"))):
        L = ctypes.CDLL(p)
        L.sincos_pairs.restype = ctypes.c_int
        L.sincos_pairs.argtypes = [ctypes.c_void_p] * 4 + [ctypes.c_size_t, ctypes.c_int, ctypes.c_void_p]
        libs[os.path.basename(p)[:-3]] = L
    cases = {"N_split": (0, False), "A_split": (1, False), "N_inter": (0, True), "A_inter": (1, True)}
    res = {k: {c_: [] for c_ in cases} for k in libs}

    def timeit(fn, reps=10):
        for _ in range(2):
            fn()
        if graph:
            reps = 20
            cap = torch.cuda.Stream()
            cap.wait_stream(torch.cuda.current_stream())
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=cap):
                for _ in range(reps):
                    fn(cap.cuda_stream)
            torch.cuda.current_stream().wait_stream(cap)
            g.replay()
            torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        if graph:
            g.replay()
        else:
            for _ in range(reps):
                fn()
        b.record()
        torch.cuda.synchronize()
        return 12 * n / (a.elapsed_time(b) / reps / 1e3) / 1e9

    for _ in range(5):
        for name, L in libs.items():
            for cname, (v, inter) in cases.items():
                if inter:
                    fn = lambda s_=st: L.sincos_pairs(th.data_ptr(), None, None, io.data_ptr(), n, v, s_)  # noqa: E731
                else:
                    fn = lambda s_=st: L.sincos_pairs(th.data_ptr(), s.data_ptr(), c.data_ptr(), None, n, v, s_)  # noqa: E731
                res[name][cname].append(timeit(fn))
    for name in libs:
        print(json.dumps({"lib": name, "n": n, "graph": graph, "GBps": {k: round(statistics.median(v), 1) for k, v in res[name].items()}}),
              flush=True)


def energy():
    """Per library and variant (N, A; split), twice alternating, after 3 s idle: 2 s of C2
    launches back to back -- board energy per launch (NVML total-energy counter), mean launch
    time over the last half, SM clock and throttle reasons at the end."""
    import time

    import pynvml
    import torch

    import inputs
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
    n = 1 << 28
    th = torch.from_numpy(inputs.generate(2, 0, n)).cuda()
    s = torch.empty(n, device="cuda")
    c = torch.empty(n, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    libs = {}
    for p in sorted(glob.glob(os.path.join(AB, "*.so"))):
        L = ctypes.CDLL(p)
        L.sincos_pairs.restype = ctypes.c_int
        L.sincos_pairs.argtypes = [ctypes.c_void_p] * 4 + [ctypes.c_size_t, ctypes.c_int, ctypes.c_void_p]
        libs[os.path.basename(p)[:-3]] = L
    out = {k: [] for k in libs}
    for _ in range(2):
        for v in (0, 1):
            for name, L in libs.items():
                go = lambda: L.sincos_pairs(th.data_ptr(), s.data_ptr(), c.data_ptr(), None, n, v, st)  # noqa: E731
                go()
                torch.cuda.synchronize()
                time.sleep(3)
                e0 = pynvml.nvmlDeviceGetTotalEnergyConsumption(h)
                t0 = time.time()
                k = 0
                evs = []
                while time.time() - t0 < 2.0:
                    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a.record()
                    for _ in range(20):
                        go()
                    b.record()
                    evs.append((a, b))
                    k += 20
                    if len(evs) > 8:
                        evs[-9][1].synchronize()
                torch.cuda.synchronize()
                mj = pynvml.nvmlDeviceGetTotalEnergyConsumption(h) - e0
                half = evs[len(evs) // 2:]
                ms = statistics.mean(a.elapsed_time(b) / 20 for a, b in half)
                out[name].append({"variant": v, "launches": k, "mJ_per_launch": round(mj / k, 2),
                                  "ms_last_half": round(ms, 4),
                                  "sm_mhz_end": pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                                  "reasons_end": hex(pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(h))})
    for name in libs:
        print(json.dumps({"lib": name, "energy": out[name]}), flush=True)


def method():
    """sincos_pairs_method with the paper's two tables (and a 3-doubling shape) on the C2 batch,
    split and interleaved, theta aligned and 1 float off: GB/s (12 B/pair), median of 5 rounds
    x 10 launches, libraries interleaved."""
    import torch

    import inputs
    import paper_cs_0406049_b200 as sp
    n = 1 << 28
    base = torch.from_numpy(inputs.generate(2, 0, n + 8)).cuda()
    s = torch.empty(n, device="cuda")
    c = torch.empty(n, device="cuda")
    io = torch.empty(2 * n, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    methods = {"paperN": sp.make_method(*sp.PAPER_METHODS[0]), "paperA": sp.make_method(*sp.PAPER_METHODS[1]),
               "deg3_3dbl": sp.make_method([1.5707963, -0.6459636, 0.0796820], [-1.2336978, 0.2536086], 3,
                                           sp.FIX_LINEAR)}
    libs = {}
    for p in sorted(glob.glob(os.path.join(AB, "*.so"))):
        L = ctypes.CDLL(p)
        L.sincos_pairs_method.restype = ctypes.c_int
        L.sincos_pairs_method.argtypes = [ctypes.c_void_p] * 4 + [ctypes.c_size_t, ctypes.c_void_p, ctypes.c_void_p]
        libs[os.path.basename(p)[:-3]] = L
    res = {k: {} for k in libs}
    for _ in range(5):
        for name, L in libs.items():
            for mname, m in methods.items():
                for inter in (False, True):
                    for off in (0, 1):
                        th = base[off:off + n]
                        outs = (None, None, io.data_ptr()) if inter else (s.data_ptr(), c.data_ptr(), None)
                        go = lambda: L.sincos_pairs_method(th.data_ptr(), *outs, n, ctypes.byref(m), st)  # noqa: E731
                        assert go() == 0
                        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                        a.record()
                        for _ in range(10):
                            go()
                        b.record()
                        torch.cuda.synchronize()
                        key = f"{mname} {'inter' if inter else 'split'} off={off}"
                        res[name].setdefault(key, []).append(12 * n / (a.elapsed_time(b) / 10 / 1e3) / 1e9)
    for name in libs:
        print(json.dumps({"lib": name, "method_GBps": {k: round(statistics.median(v), 1) for k, v in res[name].items()}}),
              flush=True)


if __name__ == "__main__":
    if sys.argv[1] == "build":
        build(sys.argv[2], sys.argv[3:])
    elif sys.argv[1] == "method":
        method()
    elif sys.argv[1] == "energy":
        energy()
    else:
        run()
