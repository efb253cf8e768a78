"""Summaries of the round's ncu evidence: launch list share per kernel, and key metrics of one --set full capture.

python tools/ncu_summary.py launches gpurun_out/launches.csv
python tools/ncu_summary.py full gpurun_out/step_full.ncu-rep
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict


def launches(path):
    rows = [r for r in csv.reader(open(path)) if r]
    hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[hdr_i]
    k, v, u = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    tot, cnt = defaultdict(float), defaultdict(int)
    for r in rows[hdr_i + 1:]:
        if len(r) <= v:
            continue
        x = float(r[v].replace(",", ""))
        x = x / 1000.0 if r[u] == "ns" else (x if r[u] == "us" else x * 1000.0)
        tot[r[k]] += x
        cnt[r[k]] += 1
    s = sum(tot.values())
    for name, t in sorted(tot.items(), key=lambda kv: -kv[1])[:10]:
        print(f"{cnt[name]:4d} x {name[:80]:80s} total {t / 1000:8.3f} ms  mean {t / cnt[name]:9.1f} us  share {100 * t / s:5.1f}%")


METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
           "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum", "launch__grid_size",
           "launch__block_size", "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic",
           "launch__shared_mem_per_block_static", "launch__occupancy_limit_registers",
           "launch__occupancy_limit_shared_mem", "smsp__sass_inst_executed_op_local_ld.sum"]


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    get = {h: (vals[i], units[i]) for i, h in enumerate(hdr)}
    print(f"Kernel Name {get['Kernel Name'][0]}")
    for m in METRICS:
        if m in get:
            print(f"{m:60s} {get[m][1]:12s} {get[m][0]}")
    stalls = sorted(((float(get[h][0].replace(',', '')), h) for h in hdr
                     if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio")
                     and get[h][0] not in ("", "n/a")), reverse=True)[:8]
    print("# top stall reasons (warps per issue-active cycle)")
    for v, h in stalls:
        print(f"{h:90s} {v:.3f}")
    def num(m):
        v, u = get[m]
        v = float(v.replace(",", ""))
        return v * {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "Tbyte": 1e12}.get(u, 1.0)
    print(f"# dram traffic per launch {num('dram__bytes_read.sum') + num('dram__bytes_write.sum'):.4e} B")


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2])
