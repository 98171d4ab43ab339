"""Parity of every tools/ab_layouts/*.so on the layouts an A/B candidate changes, before its
timings are trusted (GPU box): interleaved outputs at float offsets 0..7 and split (sin, cos)
offsets 0..7 x 0..7, theta at offsets 0 and 3, lengths around the vector / warp / span
boundaries, both variants; raw bits against the oracle and sentinel guard zones.  One JSON
line per library.
  python tools/ab_check_layouts.py"""
import ctypes
import glob
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import inputs  # noqa: E402
import oracle  # noqa: E402

AB = os.path.join(ROOT, "tools", "ab_layouts")
SENT = 0x7F8ABCDE
G = 64
NMAX = 8 * 32 * 8 * 3 + 77
LENGTHS = list(range(0, 20)) + [255, 256, 257, 8 * 32 + 9, 8 * 32 * 2 + 3, 8 * 32 * 4 - 1, 8 * 32 * 8 + 5,
                                8 * 32 * 8 * 2 + 13, NMAX]


def main():
    base = inputs.generate(2, 0, NMAX + 8)
    want = {}
    for v in (0, 1):
        s, c = oracle.sincos(base, v)
        want[v] = (torch.from_numpy(s.view(np.int32)).cuda(), torch.from_numpy(c.view(np.int32)).cuda())
    tb = torch.from_numpy(base).cuda()
    st = torch.cuda.current_stream().cuda_stream
    bi = torch.empty(2 * G + 2 * NMAX + 16, dtype=torch.int32, device="cuda")
    bs = torch.empty(2 * G + NMAX + 8, dtype=torch.int32, device="cuda")
    bc = torch.empty_like(bs)
    for p in sorted(glob.glob(os.path.join(AB, "*.so"))):
        L = ctypes.CDLL(p)
        L.sincos_pairs.restype = ctypes.c_int
        L.sincos_pairs.argtypes = [ctypes.c_void_p] * 4 + [ctypes.c_size_t, ctypes.c_int, ctypes.c_void_p]
        bad, cases = [], 0
        for v in (0, 1):
            ws, wc = want[v]
            for ot in (0, 3):
                for n in LENGTHS:
                    th = tb.data_ptr() + 4 * ot
                    for oi in range(8):
                        bi.fill_(SENT)
                        r = L.sincos_pairs(th, None, None, bi.data_ptr() + 4 * (G + oi), n, v, st)
                        got = bi[G + oi:G + oi + 2 * n]
                        ok = (r == 0 and torch.equal(got[1::2], ws[ot:ot + n]) and torch.equal(got[0::2], wc[ot:ot + n])
                              and bool((bi[:G + oi] == SENT).all()) and bool((bi[G + oi + 2 * n:] == SENT).all()))
                        cases += 1
                        if not ok:
                            bad.append(("inter", v, ot, n, oi))
                    for os_ in range(8):
                        for oc in range(8):
                            bs.fill_(SENT)
                            bc.fill_(SENT)
                            r = L.sincos_pairs(th, bs.data_ptr() + 4 * (G + os_), bc.data_ptr() + 4 * (G + oc), None,
                                               n, v, st)
                            ok = (r == 0 and torch.equal(bs[G + os_:G + os_ + n], ws[ot:ot + n]) and
                                  torch.equal(bc[G + oc:G + oc + n], wc[ot:ot + n]) and
                                  bool((bs[:G + os_] == SENT).all()) and bool((bs[G + os_ + n:] == SENT).all()) and
                                  bool((bc[:G + oc] == SENT).all()) and bool((bc[G + oc + n:] == SENT).all()))
                            cases += 1
                            if not ok:
                                bad.append(("split", v, ot, n, os_, oc))
        torch.cuda.synchronize()
        print(json.dumps({"lib": os.path.basename(p)[:-3], "cases": cases, "failing": len(bad), "first": bad[:5]}),
              flush=True)


if __name__ == "__main__":
    main()
