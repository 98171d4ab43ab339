"""Per-instruction warp-stall samples of one kernel from an ncu --set full capture (run here).

  python tools/ncu_source_summary.py REP 'sincos_vec_kernel<(int)0, (bool)0, (int)8, (int)1' OUT.txt

Groups the sampled stalls by instruction class (loads, stores, FP32 math, other) and lists
the top instructions, so the claim "the warps wait on memory, not on arithmetic" can be read
off the kernel's own SASS."""
import csv
import io
import subprocess
import sys


def main():
    rep, pat, out = sys.argv[1], sys.argv[2], sys.argv[3]
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    blocks, cur = [], None
    for line in txt.splitlines():
        if line.startswith('"Kernel Name"'):
            cur = {"name": next(csv.reader([line]))[1], "rows": []}
            blocks.append(cur)
        elif cur is not None:
            cur["rows"].append(line)
    b = next(x for x in blocks if pat in x["name"])
    rows = list(csv.DictReader(io.StringIO("\n".join(b["rows"]))))
    key = "Warp Stall Sampling (All Samples)"
    tot = sum(int(r[key] or 0) for r in rows)
    cls = {"load (LDG)": 0, "store (STG)": 0, "fp32 math (FMUL/FFMA/FADD/FRND)": 0, "other": 0}
    for r in rows:
        s, n = r["Source"].strip(), int(r[key] or 0)
        op = s.split()[0] if s else ""
        if op.startswith("@"):
            op = s.split()[1]
        if op.startswith("LDG"):
            cls["load (LDG)"] += n
        elif op.startswith("STG"):
            cls["store (STG)"] += n
        elif op.split(".")[0] in ("FMUL", "FFMA", "FADD", "FRND", "FMUL2", "FFMA2", "FADD2", "MUFU"):
            cls["fp32 math (FMUL/FFMA/FADD/FRND)"] += n
        else:
            cls["other"] += n
    stall_cols = [c for c in rows[0] if c.startswith("stall_") and "Not Issued" not in c]
    by_reason = sorted(((sum(int(r[c] or 0) for r in rows), c[6:]) for c in stall_cols), reverse=True)
    rtot = sum(v for v, _ in by_reason)
    lines = [f"kernel: {b['name']}", f"capture: {rep.split('/')[-1]}; warp-stall samples: {tot}", "",
             "samples by stall reason (long_sb = waiting on a global load's data; drain = stores",
             "draining at exit; short_sb / mio = shared/special-register queue; selected = issuing):"]
    for v, c in by_reason[:8]:
        lines.append(f"  {c:36s} {v:8d}  {v / rtot:6.1%}")
    lines += ["", "samples by the instruction the warp was stalled at (the first FMUL consumes the loaded",
              "theta, so its long_sb samples are the load latency):"]
    for k, v in cls.items():
        lines.append(f"  {k:36s} {v:8d}  {v / tot:6.1%}")
    lines += ["", "top 12 instructions by samples (stall columns as ncu names them):"]
    for r in sorted(rows, key=lambda r: -int(r[key] or 0))[:12]:
        n = int(r[key] or 0)
        top = sorted(((int(r[c] or 0), c[6:]) for c in stall_cols), reverse=True)[:2]
        lines.append(f"  {n:7d} {n / tot:6.1%}  {r['Source'].strip()[:60]:60s} "
                     + ", ".join(f"{c} {v}" for v, c in top if v))
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
