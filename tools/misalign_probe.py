"""GB/s of the hot path at theta/output offsets that do not share alignment (GPU box).
  python tools/misalign_probe.py"""
import sys, torch, json
sys.path.insert(0, '.')
import paper_cs_0406049_b200 as sp
from paper_cs_0406049_b200 import ab  # A/B build (tools only)
n = 1 << 28
base = torch.rand(n + 8, device='cuda') * 2e4 - 1e4
s = torch.empty(n + 8, device='cuda'); c = torch.empty(n + 8, device='cuda')
res = {}
for realign in (1, 2, 0):
  ab.set_realign(realign)
  for name, (to, so, co) in {'aligned': (0, 0, 0), 'theta+1': (1, 0, 0), 'out+1': (0, 1, 1), 'all+1': (1, 1, 1),
                             'theta+4': (4, 0, 0), 'sin+1 cos+2': (0, 1, 2), 'theta+3 sin+1 cos+0': (3, 1, 0)}.items():
    th, ss, cc = base[to:to + n], s[so:so + n], c[co:co + n]
    for _ in range(3): sp.sincos_pairs(th, ss, cc)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10): sp.sincos_pairs(th, ss, cc)
    b.record(); torch.cuda.synchronize()
    res[f"{name} realign={int(realign)}"] = round(12 * n / (a.elapsed_time(b) / 10 / 1e3) / 1e9, 1)
  io = torch.empty(2 * n + 8, device='cuda')
  for name, (to, oi) in {'inter theta+1': (1, 0), 'inter theta+2': (2, 0), 'inter io+1 (4-B only)': (0, 1)}.items():
    th, o = base[to:to + n], io[oi:oi + 2 * n]
    for _ in range(3): sp.sincos_pairs(th, interleaved_out=o)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10): sp.sincos_pairs(th, interleaved_out=o)
    b.record(); torch.cuda.synchronize()
    res[f"{name} realign={int(realign)}"] = round(12 * n / (a.elapsed_time(b) / 10 / 1e3) / 1e9, 1)
print(json.dumps(res))


def more():
    """16-bit outputs (8 B/pair) and the general-method kernel (12 B/pair) with theta one float
    off the outputs, re-alignment on / off."""
    out = {}
    m = sp.make_method(*sp.PAPER_METHODS[0])
    s16 = torch.empty(n, dtype=torch.float16, device='cuda'); c16 = torch.empty(n, dtype=torch.float16, device='cuda')
    for realign in (True, False):
        ab.set_realign(realign)
        for to in (0, 1):
            th = base[to:to + n]
            for name, fn, bpp in (("fp16 split", lambda: sp.sincos_pairs_dtype(th, s16, c16), 8),
                                  ("method N table split", lambda: sp.sincos_pairs_method(th, m, s[:n], c[:n]), 12)):
                for _ in range(3): fn()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                for _ in range(10): fn()
                b.record(); torch.cuda.synchronize()
                out[f"{name} theta+{to} realign={int(realign)}"] = round(bpp * n / (a.elapsed_time(b) / 10 / 1e3) / 1e9, 1)
    ab.set_realign(True)
    print(json.dumps(out))


more()
