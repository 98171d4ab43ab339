"""Key metrics of ncu captures, one block per profiled kernel (run here, no GPU needed).

  python tools/ncu_brief.py OUT.txt REP[:pairs] ...   # pairs per launch -> per-vector figures"""
import csv
import io
import subprocess
import sys

M = [("gpu__time_duration.sum", "duration"), ("dram__bytes_read.sum", "DRAM read"),
     ("dram__bytes_write.sum", "DRAM write"),
     ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
     ("sm__cycles_elapsed.avg.per_second", "SM clock"),
     ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
     ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
     ("launch__registers_per_thread", "registers / thread"), ("launch__grid_size", "grid"),
     ("launch__block_size", "block"), ("smsp__inst_executed.sum", "warp instructions"),
     ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "stall long_scoreboard / issue"),
     ("smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio", "stall short_scoreboard / issue"),
     ("smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio", "stall lg_throttle / issue"),
     ("smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio", "stall barrier / issue"),
     ("lts__t_sectors_op_write.sum", "L2 sectors written")]


def rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    h, units = r[0], r[1]
    for row in r[2:]:
        yield h, units, row


def main():
    out = [f"ncu --set full --clock-control none captures (one launch each, cold L2, serialised)\n"]
    for arg in sys.argv[2:]:
        rep, _, pairs = arg.partition(":")
        for h, units, row in rows(rep):
            d = dict(zip(h, row))
            u = dict(zip(h, units))
            out.append(f"== {rep.split('/')[-1]}: {d.get('Kernel Name', '')}")
            for k, name in M:
                if k in d:
                    out.append(f"   {name:34s} {d[k]:>18s} {u.get(k, '')}")
            if pairs and "smsp__inst_executed.sum" in d:
                n = int(eval(pairs))
                wi = float(d["smsp__inst_executed.sum"].replace(",", ""))
                out.append(f"   {'warp instructions / 256 pairs':34s} {wi / (n / 256):18.1f}")
                dur = float(d["gpu__time_duration.sum"].replace(",", ""))
                scale = {"ms": 1e-3, "us": 1e-6, "ns": 1e-9}.get(u.get("gpu__time_duration.sum", "us"), 1e-6)
                out.append(f"   {'pairs / s':34s} {n / (dur * scale):18.4g}")
            out.append("")
    open(sys.argv[1], "w").write("\n".join(out))
    print("\n".join(out))


if __name__ == "__main__":
    main()
