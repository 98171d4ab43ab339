"""GPU pairs against long-double sinl/cosl (SURVEY 8(d) error measurement; GPU box, host CPU
for the reference): C1-C3 on every element, C4/C5 on every 64th element (the kernel's output
for an element depends only on its angle, so the subsample's angles are evaluated directly).
Also the oracle's own error on the same elements -- equal, the outputs being bit-identical.
Prints one JSON line per (config, variant).   python tools/error_longdouble.py"""
import json
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import inputs  # noqa: E402
import oracle  # noqa: E402
import paper_cs_0406049_b200 as sp  # noqa: E402

CONFIGS = {1: (1 << 20, 1), 2: (1 << 28, 1), 3: (1 << 24, 1), 4: (1 << 30, 64), 5: (1 << 32, 64)}


def stats(theta, s, c, ref, threads):
    chunk = 1 << 20
    spans = [(i, min(i + chunk, theta.size)) for i in range(0, theta.size, chunk)]
    with ThreadPoolExecutor(threads) as ex:
        parts = list(ex.map(lambda ab: oracle.error_stats(theta[ab[0]:ab[1]], s[ab[0]:ab[1]], c[ab[0]:ab[1]], ref),
                            spans))
    n = sum(p.count for p in parts)
    return {"n": n, "nan": sum(p.nan_count for p in parts), "max_comb": max(p.max_comb for p in parts),
            "rms": (sum(p.sum_sq for p in parts) / n) ** 0.5 if n else 0.0,
            "max_amp": max(p.max_amp for p in parts)}


def main():
    threads = os.cpu_count() or 1
    for cfg, (n, stride) in CONFIGS.items():
        if stride == 1:
            th = inputs.generate(cfg, 0, n)
        else:
            th = inputs.generate_at(cfg, np.arange(0, n, stride, dtype=np.uint64))
        t = torch.from_numpy(th).cuda()
        for v in (0, 1):
            t0 = time.time()
            s, c = sp.sincos(t, variant=v)
            gs, gc = s.cpu().numpy(), c.cpu().numpy()
            os_ = np.empty_like(th)
            oc = np.empty_like(th)
            spans = [(i, min(i + (1 << 22), th.size)) for i in range(0, th.size, 1 << 22)]
            with ThreadPoolExecutor(threads) as ex:
                list(ex.map(lambda ab: oracle.sincos_into(th[ab[0]:ab[1]], os_[ab[0]:ab[1]], oc[ab[0]:ab[1]], v),
                            spans))
            same = bool(np.all((gs == os_) | (np.isnan(gs) & np.isnan(os_))) and
                        np.all((gc == oc) | (np.isnan(gc) & np.isnan(oc))))
            line = {"config": f"C{cfg}", "variant": "NA"[v], "elements": int(th.size),
                    "sample": "all" if stride == 1 else f"every {stride}th of {n}",
                    "gpu_equals_oracle": same,
                    "gpu_vs_long_double": stats(th, gs, gc, oracle.REF_LONGDOUBLE, threads),
                    "oracle_vs_long_double": stats(th, os_, oc, oracle.REF_LONGDOUBLE, threads),
                    "gpu_vs_double": stats(th, gs, gc, oracle.REF_DOUBLE, threads),
                    "seconds": round(time.time() - t0, 1), "host_threads": threads}
            print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
