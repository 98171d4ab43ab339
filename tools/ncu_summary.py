"""Summarise ncu output into profiles/ (run here, no GPU needed).

  python tools/ncu_summary.py --rep gpurun_out/prof_r01.ncu-rep --launches gpurun_out/launches_r01.csv \
      --n 268435456 --tag r01

Writes profiles/ncu_<tag>_summary.txt (key metrics per profiled launch, the launch list
with each kernel's share of the step) and profiles/ncu_summary.json (per-launch DRAM
bytes of the dominant kernel, read by bench.py for roofline.traffic).
"""
import argparse
import csv
import io
import json
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("dram__cycles_elapsed.avg.per_second", "DRAM clock"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("sm__inst_issued.avg.pct_of_peak_sustained_active", "issue slots busy %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active", "FMA-heavy pipe %"),
    ("sm__pipe_fmalite_cycles_active.avg.pct_of_peak_sustained_active", "FMA-lite pipe %"),
    ("sm__inst_executed_pipe_fmaheavy.sum", "FMA-heavy warp instructions"),
    ("sm__inst_executed_pipe_fmalite.sum", "FMA-lite warp instructions"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe %"),
    ("sm__pipe_xu_cycles_active.avg.pct_of_peak_sustained_active", "XU pipe %"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "stall long_scoreboard / issue"),
    ("smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio", "stall lg_throttle / issue"),
    ("smsp__average_warps_issue_stalled_drain_per_issue_active.ratio", "stall drain / issue"),
    ("smsp__average_warps_issue_stalled_wait_per_issue_active.ratio", "stall wait / issue"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("launch__registers_per_thread", "registers / thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("lts__t_sectors_srcunit_tex_op_read.sum", "L2 sectors read (from SM)"),
    ("lts__t_sectors_srcunit_tex_op_write.sum", "L2 sectors written (from SM)"),
]


def raw_rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    return hdr, units, data


def to_float(s):
    try:
        return float(s.replace(",", ""))
    except ValueError:
        return None


def scale(v, unit):
    """Convert ncu's unit to base units (bytes, seconds, Hz)."""
    f = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "ns": 1e-9, "us": 1e-6,
         "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "nsecond": 1e-9, "Ghz": 1e9, "Mhz": 1e6, "hz": 1,
         "cycle/second": 1, "cycle/nsecond": 1e9, "cycle/usecond": 1e6}.get(unit, 1)
    return v * f


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rep", required=True)
    ap.add_argument("--launches", default=None)
    ap.add_argument("--n", type=int, required=True, help="elements per launch of the profiled kernels")
    ap.add_argument("--tag", required=True)
    args = ap.parse_args()
    hdr, units, data = raw_rows(args.rep)
    col = {h: i for i, h in enumerate(hdr)}
    lines = [f"ncu --set full --clock-control none capture: {os.path.basename(args.rep)}; elements per launch n = {args.n}",
             f"algorithmic bytes per launch = 12 n = {12 * args.n} (4 B theta in, 8 B sin+cos out)", ""]
    kernels = []
    for d in data:
        name = d[col["Kernel Name"]]
        k = {"kernel": name}
        lines.append(f"== {name}")
        for m, label in METRICS:
            if m not in col:
                continue
            raw = d[col[m]]
            lines.append(f"   {label:34s} {raw:>18s} {units[col[m]]}")
            v = to_float(raw)
            if v is not None:
                k[m] = scale(v, units[col[m]])
        rb, wb = k.get("dram__bytes_read.sum"), k.get("dram__bytes_write.sum")
        if rb is not None and wb is not None:
            t = k.get("gpu__time_duration.sum")
            lines.append(f"   {'DRAM bytes / algorithmic bytes':34s} {(rb + wb) / (12 * args.n):18.4f}")
            if t:
                lines.append(f"   {'DRAM GB/s under ncu (cold, serial)':34s} {(rb + wb) / t / 1e9:18.1f}")
        lines.append("")
        kernels.append(k)
    if args.launches and os.path.exists(args.launches):
        rows = [r for r in csv.reader(open(args.launches)) if len(r) > 10 and r[0] != "ID" and not r[0].startswith("==")]
        tot = {}
        for r in rows:
            if r[-3] == "gpu__time_duration.sum":
                nm = r[4].split("(")[0] + " grid " + r[8].strip("()").split(",")[0]
                tot.setdefault(nm, []).append(scale(float(r[-1].replace(",", "")), r[-2]))
        all_t = sum(sum(v) for v in tot.values())
        # the hot path's step: variant N and A of the bench launch (the largest grid of each)
        step = {}
        for nm, v in tot.items():
            for var in ("0", "1"):
                if f"sincos_vec_kernel<{var}, 0, 8, 1, 1, 0>" in nm or f"sincos_vec_kernel<{var}, 1, 8, 1, 1, 0>" in nm:
                    g = int(nm.rsplit(" ", 1)[1])
                    if var not in step or g > step[var][0]:
                        step[var] = (g, nm, v)
        if step:
            st = sum(sum(x[2]) / len(x[2]) for x in step.values())
            lines.append("== the hot path's step under ncu (one launch per variant, mean launch time)")
            for var, (g, nm, v) in sorted(step.items()):
                m = sum(v) / len(v)
                lines.append(f"   variant {'NA'[int(var)]}: {nm:60s} launches {len(v):4d}  mean {1e6 * m:9.1f} us"
                             f"  share of step {m / st:6.1%}  GB/s {12 * args.n / m / 1e9:8.1f}")
            lines.append("")
        lines.append("== launch list of the whole command (ncu --metrics gpu__time_duration.sum, cold-cache, "
                     "serialised), by kernel and grid size; includes the untimed legs (ceiling, stats, e2e "
                     "chunks, NEXT-row measurements)")
        for nm, v in sorted(tot.items(), key=lambda kv: -sum(kv[1])):
            lines.append(f"   {nm:70s} launches {len(v):4d}  mean {1e6 * sum(v) / len(v):9.1f} us  share {sum(v) / all_t:6.1%}")
    txt = os.path.join(ROOT, "profiles", f"ncu_{args.tag}_summary.txt")
    open(txt, "w").write("\n".join(lines) + "\n")
    # the dominant (longest) sincos kernel's per-launch DRAM traffic, for bench.py
    sk = [k for k in kernels if "sincos_vec_kernel" in k["kernel"] and "dram__bytes_read.sum" in k]
    if sk:
        # the bench's kernel (variant N, split, 256-bit, U = 1, the default launch) if captured,
        # else the longest sincos kernel
        bench_k = [k for k in sk if "sincos_vec_kernel<0, 0, 8, 1, 1, 0>" in k["kernel"]]
        dom = bench_k[0] if bench_k else max(sk, key=lambda k: k.get("gpu__time_duration.sum", 0))
        js = {"tag": args.tag, "rep": os.path.basename(args.rep),
              "dominant": {"kernel": dom["kernel"], "n": args.n, "dram_bytes_read": dom["dram__bytes_read.sum"],
                           "dram_bytes_write": dom["dram__bytes_write.sum"],
                           "duration_s_under_ncu": dom.get("gpu__time_duration.sum")},
              "all": [{"kernel": k["kernel"], "dram_bytes_read": k.get("dram__bytes_read.sum"),
                       "dram_bytes_write": k.get("dram__bytes_write.sum")} for k in sk]}
        path = os.path.join(ROOT, "profiles", "ncu_summary.json")
        if os.path.exists(path):          # keep the per-config DRAM captures (tools/prof_configs.py)
            prev = json.load(open(path))
            for k in ("by_config", "by_config_source"):
                if k in prev and k not in js:
                    js[k] = prev[k]
        json.dump(js, open(path, "w"), indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
