"""split <-> interleaved fp32 adapters at shared and unshared pointer offsets (floats), C2 size,
GB/s of 16 B moved per element (GPU box).  One JSON line per layout.
  python tools/adapter_offsets_probe.py"""
import json, statistics, torch, sys
sys.path.insert(0, '.')
import paper_cs_0406049_b200 as sp
N = 1 << 28
def timed(fn):
    for _ in range(3): fn()
    ms = []
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(4): fn()
        b.record(); torch.cuda.synchronize(); ms.append(a.elapsed_time(b) / 4)
    return round(16 * N / (statistics.median(ms) / 1e3) / 1e9, 1)
s = torch.rand(N + 16, device='cuda'); c = torch.rand(N + 16, device='cuda'); io = torch.empty(2 * N + 16, device='cuda')
for os_, oc, oi in ((0, 0, 0), (1, 1, 2), (0, 1, 0), (0, 0, 2), (1, 2, 4)):   # interleaved: 8-B aligned pairs (ABI)
    r = {"sin+": os_, "cos+": oc, "inter+": oi}
    r["interleave_GBps"] = timed(lambda: sp.interleave(s[os_:os_ + N], c[oc:oc + N], interleaved_out=io[oi:oi + 2 * N]))
    r["deinterleave_GBps"] = timed(lambda: sp.deinterleave(io[oi:oi + 2 * N], s[os_:os_ + N], c[oc:oc + N]))
    print(json.dumps(r), flush=True)
