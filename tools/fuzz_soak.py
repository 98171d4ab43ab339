"""Long seeded random soak of every pair entry point against the oracle (GPU box; evidence, not
a test): random lengths (0 .. 300k), element offsets of theta and each output, layouts,
variants, entry points (sincos_pairs, _dtype fp32, _method with the paper's table, phase grid
with f = [1], the batched call with several arrays), launch configurations, re-alignment and
PDL switches, input generators.  Runs for --seconds, prints one JSON line of counts.
  python tools/fuzz_soak.py --seconds 300"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import inputs  # noqa: E402
import oracle  # noqa: E402
import paper_cs_0406049_b200 as sp  # noqa: E402
from paper_cs_0406049_b200 import ab  # A/B build (tools only)
from helpers import same_values  # noqa: E402


def draw_theta(rng, n):
    kind = rng.integers(0, 7)
    if kind < 5:
        return inputs.generate(int(kind) + 1, int(rng.integers(0, 1 << 20)), n)
    if kind == 5:
        return rng.integers(0, 1 << 32, n, dtype=np.uint64).astype(np.uint32).view(np.float32)
    return rng.uniform(-1e6, 1e6, n).astype(np.float32)


def one_case(rng):
    r = rng.random()
    n = int(rng.integers(0, 40)) if r < 0.3 else int(rng.integers(40, 5000)) if r < 0.8 \
        else int(rng.integers(5000, 300_000))
    variant = int(rng.integers(0, 2))
    inter = bool(rng.integers(0, 2))
    entry = ["pairs", "dtype32", "method", "phase", "batched", "fp16", "bf16", "phase2d"][int(rng.integers(0, 8))]
    if entry == "phase2d":                # an nf x nt grid: theta_ij = RN(f_i t_j), the fp32 products
        if rng.random() < 0.5:            # many short rows: the tiny / staged / short-row kernels' regions
            nt2 = int(rng.integers(1, 16))
            nf2 = max(1, n // nt2)
        else:
            nf2 = int(rng.integers(1, 24))
            nt2 = max(1, n // nf2)
        f2 = rng.uniform(-50, 50, nf2).astype(np.float32)
        toff2 = int(rng.integers(0, 8))
        t2 = draw_theta(rng, nt2 + 8)[toff2:toff2 + nt2]
        n = nf2 * nt2
        with np.errstate(over="ignore", invalid="ignore"):   # inf / NaN products are inputs too
            th = (f2[:, None] * t2[None, :]).astype(np.float32).ravel()
    else:
        th = draw_theta(rng, n)
    ot, os_, oc = (int(x) for x in rng.integers(0, 8, 3))
    if rng.random() < 0.5:
        oc = os_
    cfg = [(128, 0, 8, 1, 0), (256, 0, 8, 2, 0), (512, 4, 4, 1, 1), (128, 1, 8, 4, 0)][int(rng.integers(0, 4))]
    if entry == "batched" or rng.random() < 0.5:
        # the A/B build (the batched entry exists only there), with a random launch shape,
        # re-alignment and PDL switch
        ab.set_launch_config(*cfg)
        ab.set_realign(bool(rng.random() < 0.85))
        ab.set_pdl(bool(rng.random() < 0.7))
    else:
        ab.use(False)                     # the product library: its one configuration
        cfg = "product"
    tbuf = torch.empty(n + 16, dtype=torch.float32, device="cuda")
    tbuf[ot:ot + n].copy_(torch.from_numpy(th))
    t = tbuf[ot:ot + n]
    dt = {"fp16": torch.float16, "bf16": torch.bfloat16}.get(entry, torch.float32)
    if inter:
        io = torch.empty(2 * n + 16, dtype=dt, device="cuda")[2 * os_ if dt != torch.float32 else os_:][:2 * n]
        outs = {"interleaved_out": io}
    else:
        outs = {"sin_out": torch.empty(n + 16, dtype=dt, device="cuda")[os_:os_ + n],
                "cos_out": torch.empty(n + 16, dtype=dt, device="cuda")[oc:oc + n]}
    if entry == "pairs":
        sp.sincos_pairs(t, variant=variant, **outs)
    elif entry == "dtype32":
        sp.sincos_pairs_dtype(t, variant=variant, **outs)
    elif entry == "method":
        sp.sincos_pairs_method(t, sp.make_method(*sp.PAPER_METHODS[variant]), **outs)
    elif entry in ("fp16", "bf16"):
        sp.sincos_pairs_dtype(t, variant=variant, **outs)
    elif entry == "phase":
        sp.phase_grid(torch.ones(1, device="cuda"), t, units=sp.RADIANS, variant=variant, **outs)
    elif entry == "phase2d":
        tb2 = torch.empty(nt2 + 8, device="cuda")
        tb2[toff2:toff2 + nt2].copy_(torch.from_numpy(t2))
        sp.phase_grid(torch.from_numpy(f2).cuda(), tb2[toff2:toff2 + nt2], units=sp.RADIANS, variant=variant, **outs)
    else:
        if inter:
            ab.sincos_pairs_batched([t, t[: n // 2]], interleaved_outs=[io, torch.empty(2 * (n // 2), device="cuda")],
                                    variant=variant)
        else:
            ab.sincos_pairs_batched([t], [outs["sin_out"]], [outs["cos_out"]], variant=variant)
    torch.cuda.synchronize()
    if inter:
        v = outs["interleaved_out"].float().cpu().numpy()
        gs, gc = v[1::2], v[0::2]
    else:
        gs, gc = outs["sin_out"].float().cpu().numpy(), outs["cos_out"].float().cpu().numpy()
    ws, wc = oracle.sincos(th, variant)
    if dt != torch.float32:               # the library's RN cast of the oracle's fp32 pair
        ws = torch.from_numpy(ws).to(dt).float().numpy()
        wc = torch.from_numpy(wc).to(dt).float().numpy()
    ok = bool(same_values(gs, ws).all() and same_values(gc, wc).all())
    return ok, n, entry


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seconds", type=float, default=300)
    ap.add_argument("--seed", type=int, default=20261020)
    args = ap.parse_args()
    rng = np.random.default_rng(args.seed)
    t0 = time.time()
    cases = elements = bad = 0
    by_entry = {}
    first_bad = None
    while time.time() - t0 < args.seconds:
        ok, n, entry = one_case(rng)
        cases += 1
        elements += n
        by_entry[entry] = by_entry.get(entry, 0) + 1
        if not ok:
            bad += 1
            first_bad = first_bad or cases
    ab.set_launch_config()
    ab.set_realign(True)
    ab.set_pdl(True)
    print(json.dumps({"cases": cases, "elements": elements, "mismatching_cases": bad, "first_bad_case": first_bad,
                      "by_entry": by_entry, "seconds": round(time.time() - t0, 1), "seed": args.seed}))


if __name__ == "__main__":
    main()
