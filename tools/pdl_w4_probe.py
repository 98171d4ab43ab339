import sys, json, torch
sys.path.insert(0, '.')
import paper_cs_0406049_b200 as sp
from paper_cs_0406049_b200 import ab  # A/B build (tools only)
n = 1 << 28
base = torch.rand(n + 8, device='cuda') * 2e4 - 1e4
s = torch.empty(n, device='cuda'); c = torch.empty(n, device='cuda')
res = {}
for rep in range(2):
  for pdl in (False, True):
    ab.set_pdl(pdl)
    for name, to in (('aligned', 0), ('theta+4', 4)):
        th = base[to:to + n]
        for _ in range(3): sp.sincos_pairs(th, s, c)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(10): sp.sincos_pairs(th, s, c)
        b.record(); torch.cuda.synchronize()
        res.setdefault(f"{name} pdl={int(pdl)}", []).append(round(12 * n / (a.elapsed_time(b) / 10 / 1e3) / 1e9, 1))
print(json.dumps(res))
