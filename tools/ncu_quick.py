"""Print the key metrics and top stall/instruction lines of an ncu report (read here, no GPU)."""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "launch__registers_per_thread", "lts__t_sector_hit_rate.pct",
        "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_branch_resolving_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_drain_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_membar_per_issue_active.ratio",
        "nvlrx__bytes.sum", "nvltx__bytes.sum"]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def main(rep, ntop=25):
    h, u, data = raw(rep)
    for d in data:
        for k in KEYS:
            if k in h:
                i = h.index(k)
                print(f"{k:80s} {d[i]} {u[i]}")
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hh = rows[1]
    body = rows[2:]
    iA, iS, iW, iI = hh.index("Address"), hh.index("Source"), hh.index("Warp Stall Sampling (All Samples)"), \
        hh.index("Instructions Executed")
    tot = sum(int(r[iI] or 0) for r in body)
    print("instructions", tot)
    for r in sorted(body, key=lambda r: -int(r[iI] or 0))[:ntop]:
        print(r[iI], r[iW], r[iA][-5:], r[iS][:90])


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
