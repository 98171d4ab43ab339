import sys, time, ctypes, torch
sys.path.insert(0, '.')
import paper_cs_0406049_b200 as sp
from paper_cs_0406049_b200 import ab  # A/B build (tools only)
count, n = 1000, 4096
base = torch.rand(count * n, device="cuda")
s, c = torch.empty_like(base), torch.empty_like(base)
ts = [base[i*n:(i+1)*n] for i in range(count)]; ss = [s[i*n:(i+1)*n] for i in range(count)]; cs = [c[i*n:(i+1)*n] for i in range(count)]
table = ab.BatchTable(ts, ss, cs)
L = ab.lib(); st = torch.cuda.current_stream().cuda_stream
def raw(): L.sincos_pairs_batched(table.tab.ctypes.data, count, 0, st)
def host_us(fn, k=200):
    for _ in range(5): fn()
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(k): fn()
    t1 = time.perf_counter(); torch.cuda.synchronize(); t2 = time.perf_counter()
    return 1e6*(t1-t0)/k, 1e6*(t2-t0)/k
print("raw host/total us", host_us(raw))
print("run host/total us", host_us(table.run))
