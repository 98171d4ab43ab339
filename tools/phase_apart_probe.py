"""sincos_phase_grid with unshared output alignment (split cos[] off sin[]'s 32-B offset,
interleaved pairs only 4-B aligned) beside the aligned layouts, turns, variant N, ~2^30 pairs
per launch, rows of 2^15 / 1001 / 5 pairs (GPU box).  One JSON line per case.
  python tools/phase_apart_probe.py"""
import json, statistics, torch, sys
sys.path.insert(0, '.')
import paper_cs_0406049_b200 as sp
dev = torch.device('cuda:0')
def timed(fn):
    for _ in range(3): fn()
    ms = []
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(4): fn()
        b.record(); torch.cuda.synchronize(); ms.append(a.elapsed_time(b) / 4)
    return statistics.median(ms)
sb = torch.empty((1 << 30) + 64, device=dev); cb = torch.empty((1 << 30) + 64, device=dev); ib = torch.empty((1 << 31) + 64, device=dev)
for nt in (1 << 15, 1001, 5):
    nf = (1 << 30) // nt
    f = torch.rand(nf, device=dev) * 512; t = torch.rand(nt, device=dev)
    n = nf * nt
    for name, kw in (("split aligned", dict(sin_out=sb[:n], cos_out=cb[:n])),
                     ("split cos+1", dict(sin_out=sb[:n], cos_out=cb[1:1 + n])),
                     ("split cos+4", dict(sin_out=sb[:n], cos_out=cb[4:4 + n])),
                     ("inter+0", dict(interleaved_out=ib[:2 * n])),
                     ("inter+1", dict(interleaved_out=ib[1:1 + 2 * n]))):
        ms = timed(lambda: sp.phase_grid(f, t, units=sp.TURNS, **kw))
        print(json.dumps({"nt": nt, "case": name, "GBps_written": round(8 * n / (ms / 1e3) / 1e9, 1)}), flush=True)
