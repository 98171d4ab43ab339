import sys, json, torch
sys.path.insert(0, '.')
import paper_cs_0406049_b200 as sp
n = 1 << 28
s = torch.rand(n, device='cuda'); c = torch.rand(n, device='cuda'); io = torch.empty(2 * n, device='cuda')
def t(fn, reps=10):
    for _ in range(3): fn()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps): fn()
    b.record(); torch.cuda.synchronize()
    return 16 * n / (a.elapsed_time(b) / reps / 1e3) / 1e9
print(json.dumps({"interleave_GBps": round(t(lambda: sp.interleave(s, c, io)), 1),
                  "deinterleave_GBps": round(t(lambda: sp.deinterleave(io, s, c)), 1),
                  "torch_stack_GBps": round(t(lambda: torch.stack((c, s), dim=1, out=io.view(n, 2))), 1)}))
