"""Summarise an ncu report (run here, no GPU): per-kernel key metrics and the
hottest SASS lines.  python tools/ncu_summary.py rep.ncu-rep [--src N] [--kernel REGEX]"""
import csv
import io
import subprocess
import sys

KEYS = [("gpu__time_duration.sum", "us"), ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor%"),
        ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram%"), ("dram__bytes_read.sum", "rdMB"),
        ("dram__bytes_write.sum", "wrMB"), ("smsp__inst_executed.sum", "inst"),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue%"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ%"),
        ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "st_lsb"),
        ("smsp__average_warps_issue_stalled_wait_per_issue_active.ratio", "st_wait"),
        ("smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio", "st_bar"),
        ("smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio", "st_ssb"),
        ("smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio", "st_mio"),
        ("smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio", "st_math"),
        ("launch__grid_size", "grid"), ("launch__registers_per_thread", "regs")]


def run(args):
    return subprocess.run(["ncu", "-i", *args], capture_output=True, text=True).stdout


def main():
    rep = sys.argv[1]
    nsrc = int(sys.argv[sys.argv.index("--src") + 1]) if "--src" in sys.argv else 0
    rows = list(csv.reader(io.StringIO(run([rep, "--page", "raw", "--csv"]))))
    hdr = rows[0]
    idx = {h: i for i, h in enumerate(hdr)}
    print("kernel".ljust(34) + "".join(k[1].rjust(9) for k in KEYS))
    for r in rows[2:]:
        name = r[idx["Kernel Name"]][:33]
        vals = []
        for k, _ in KEYS:
            v = r[idx[k]] if k in idx else ""
            try:
                f = float(v)
                vals.append((f"{f:.3g}" if f < 1e6 else f"{f / 1e6:.1f}M").rjust(9))
            except ValueError:
                vals.append(v[:8].rjust(9))
        print(name.ljust(34) + "".join(vals))
    if nsrc:
        out = run([rep, "--page", "source", "--csv", "--print-source", "sass"])
        blocks, cur = [], None
        hdr2 = None
        for r in csv.reader(io.StringIO(out)):
            if r and r[0] == "Kernel Name":
                cur = [r[1], []]
                blocks.append(cur)
                continue
            if r and r[0] == "Address":
                hdr2 = r
                continue
            if r and r[0].startswith("0x") and cur is not None:
                cur[1].append(r)
        if hdr2 is None:
            return
        iS = hdr2.index("Warp Stall Sampling (All Samples)")
        iE = hdr2.index("Instructions Executed")
        iSrc = hdr2.index("Source")
        for name, data in blocks:
            tot = sum(int(x[iS] or 0) for x in data)
            print(f"\n== {name[:80]}  samples={tot}")
            top = sorted(range(len(data)), key=lambda i: -int(data[i][iS] or 0))[:nsrc]
            for i in sorted(top):
                print(f"{i:6d} {data[i][iS]:>6} {data[i][iE]:>9}  {data[i][iSrc][:80]}")


if __name__ == "__main__":
    main()
