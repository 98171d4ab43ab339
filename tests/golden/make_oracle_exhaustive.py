"""Whole-input-space runs of the ORACLE (calls only oracle/; nothing from the CUDA path).

Writes tests/golden/oracle_exhaustive.json:
  * kernel-only maxima over every fp32 q in [0, 1/2]        (SURVEY [X5])
  * end-to-end maxima over every fp32 theta in [+0, fl32(pi)] (SURVEY [X5])
  * the all-2^32 transcription hash, NaN and exact-(0,1) counts (SURVEY [X13])
for variants N, A and A-text.  tests/test_oracle_pins.py compares this file with
the survey's independent transcription (tests/golden/survey_crosscheck.json);
the GPU all-bit-patterns test compares the CUDA path's hash with it.

Usage: python tests/golden/make_oracle_exhaustive.py [--threads T]
(about 15 CPU-minutes per variant on one core).
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..", "..")))
import oracle  # noqa: E402

Q_HALF = 0x3F000000      # fp32 bits of 0.5
FL32_PI = 0x40490FDB     # fp32 bits of fl32(pi)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--threads", type=int, default=0)
    ap.add_argument("--out", default=os.path.join(os.path.dirname(__file__), "oracle_exhaustive.json"))
    args = ap.parse_args()
    res = {"_source": "written by tests/golden/make_oracle_exhaustive.py (oracle/ only)"}
    for name, v in (("N", oracle.VARIANT_N), ("A", oracle.VARIANT_A), ("A_text", oracle.VARIANT_A_TEXT)):
        r = {}
        t0 = time.time()
        st = oracle.sweep_bits(v, 1, 0, Q_HALF, args.threads)
        r["q_half"] = {"max": st.max_comb, "argmax": st.worst_x, "argmax_bits": hex(st.worst_bits),
                       "max_amp": st.max_amp, "count": st.count, "rms": st.rms}
        st = oracle.sweep_bits(v, 0, 0, FL32_PI, args.threads)
        r["theta_0_pi"] = {"max": st.max_comb, "argmax": st.worst_x, "argmax_bits": hex(st.worst_bits),
                           "max_amp": st.max_amp, "count": st.count, "rms": st.rms}
        h, nn, ex = oracle.hash_bits(v, 0, 0xFFFFFFFF, args.threads)
        r["all_bits"] = {"hash": "0x%016X" % h, "nan_pairs": nn, "exact_0_1": ex}
        r["seconds"] = time.time() - t0
        res[name] = r
        print(name, json.dumps(r), flush=True)
    with open(args.out, "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
