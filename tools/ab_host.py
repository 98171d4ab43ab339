"""A/B of libraries on the host-buffer pipeline (sincos_pairs_host; tuning aid, GPU box): the
bench's e2e step -- 2^28 angles, both variants, split outputs, pinned host buffers, a 256 MiB
workspace -- for every tools/ab_host/*.so (rotating order each round), beside the PCIe roofline
of the same buffers (bench.pcie_roofline).  One JSON line."""
import ctypes
import glob
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import bench
    n = 1 << 28
    libs = {}
    for p in sorted(glob.glob(os.environ.get("AB_HOST_GLOB", os.path.join(ROOT, "tools", "ab_host", "*.so")))):
        L = ctypes.CDLL(p)
        L.sincos_pairs_host.restype = ctypes.c_int
        L.sincos_pairs_host.argtypes = [ctypes.c_void_p] * 4 + [ctypes.c_size_t, ctypes.c_int, ctypes.c_void_p,
                                                                ctypes.c_size_t, ctypes.c_void_p]
        libs[os.path.basename(p)[:-3]] = L
    dev = torch.device("cuda", 0)
    th = (torch.rand(n) * 2e4 - 1e4).pin_memory()
    so, co = torch.empty(n).pin_memory(), torch.empty(n).pin_memory()
    ws = torch.empty(int(os.environ.get("AB_WS_MIB", "256")) << 20, dtype=torch.uint8, device=dev)
    st = torch.cuda.current_stream().cuda_stream

    def step(L):
        for v in (0, 1):
            r = L.sincos_pairs_host(th.data_ptr(), so.data_ptr(), co.data_ptr(), None, n, v, ws.data_ptr(),
                                    ws.numel(), st)
            assert r == 0, r

    res = {k: [] for k in libs}
    order = list(libs)
    for rnd in range(len(order) * -(-int(os.environ.get("AB_ROUNDS", "12")) // len(order))):
        for name in order[rnd % len(order):] + order[:rnd % len(order)]:
            step(libs[name])
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
            ev[0].record()
            for k in range(3):
                step(libs[name])
                ev[k + 1].record()
            torch.cuda.synchronize()
            res[name] += [ev[k].elapsed_time(ev[k + 1]) for k in range(3)]
    # every library's outputs equal the first one's (variant A, the last step's)
    same = {}
    ref = None
    for name in order:
        step(libs[name])
        torch.cuda.synchronize()
        got = (so.clone(), co.clone())
        if ref is None:
            ref = got
        same[name] = bool(torch.equal(got[0].view(torch.int32), ref[0].view(torch.int32)) and
                          torch.equal(got[1].view(torch.int32), ref[1].view(torch.int32)))
    roof = bench.pcie_roofline(th, n, 2, dev, [so, co])
    print(json.dumps({"ws_mib": ws.numel() >> 20, "ms_per_step_median": {k: statistics.median(v) for k, v in res.items()},
                      "ms_per_step_min": {k: min(v) for k, v in res.items()},
                      "roofline_concurrent_ms": roof["concurrent_ms"],
                      "frac": {k: roof["step_floor_ms"] / statistics.median(v) for k, v in res.items()},
                      "outputs_equal_first": same}))


if __name__ == "__main__":
    main()
