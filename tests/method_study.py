"""NEXT(3) design study (test-side script; uses the oracle): kernel-only accuracy of regenerated
methods over fp32 q in [0, 1/2] (every 31st pattern) for doubling counts 1..4, series degrees
and both fitting methods, with the FP32-pipe op count per pair of each method.

  python tests/method_study.py  ->  profiles/method_study_r01.json
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from paper_cs_0406049_b200 import coeff_fit as cf  # noqa: E402


def ops(n_ss, n_cc, n, kind):
    """FP32-pipe ops per pair: scale, round+sub (2), q^2, Horner (n_ss - 1 + n_cc FFMA) + the
    s multiply, c's final FFMA if n_cc, per doubling 4 (c^2, fma, s*c, *2), fix 2 (N) or
    2 + MUFU (A), apply 2."""
    return 1 + 2 + 1 + (n_ss - 1) + 1 + n_cc + 4 * n + 2 + 2


def main():
    rows = []
    for n in (1, 2, 3, 4):
        for ds, dc in ((3, 2), (3, 3), (4, 3), (5, 4), (6, 5)):
            for kind in ("normalized", "angle"):
                f = cf.fit_normalized(n, ds, dc, weight="relative") if kind == "normalized" else cf.fit_angle(n, ds, dc)
                ss, cc = f.fp32()
                fix = oracle.FIX_LINEAR_PENULTIMATE if kind == "normalized" else oracle.FIX_RECIPROCAL
                st = oracle.method_sweep_q(oracle.make_method(ss, cc, n, fix), stride=31)
                rows.append({"doublings": n, "n_ss": ds, "n_cc": dc, "fit": kind, "max_err": st.max_comb,
                             "rms_err": st.rms, "max_amp": st.max_amp, "fp32_ops_per_pair": ops(ds, dc, n, kind)})
                print(json.dumps(rows[-1]), flush=True)
    for v, name in ((oracle.VARIANT_N, "paper N"), (oracle.VARIANT_A, "paper A")):
        st = oracle.method_sweep_q(oracle.paper_method(v), stride=31)
        rows.append({"doublings": 2, "n_ss": 4, "n_cc": 3, "fit": name, "max_err": st.max_comb, "rms_err": st.rms,
                     "max_amp": st.max_amp, "fp32_ops_per_pair": ops(4, 3, 2, name)})
    out = os.path.join(ROOT, "profiles", "method_study_r01.json")
    json.dump({"_source": "tests/method_study.py (oracle + coeff_fit); kernel-only error over every 31st fp32 "
                          "q in [0, 1/2]", "rows": rows}, open(out, "w"), indent=1)


if __name__ == "__main__":
    main()
