"""Summaries of ncu captures for profiles/:
  python tools/ncu_summary.py launches <launches.csv>        per-kernel time shares
  python tools/ncu_summary.py full <report.ncu-rep> [id]     key --set full metrics per launch
"""
import csv
import subprocess
import sys
from collections import defaultdict

KEYS = [
    "gpu__time_duration.sum", "launch__grid_size", "launch__block_size",
    "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.per_cycle_active", "sm__warps_active.avg.per_cycle_active",
    "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sectors.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__average_warp_latency_issue_stalled_long_scoreboard",
]


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr, agg = None, defaultdict(lambda: [0, 0.0])
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") != "gpu__time_duration.sum":
                continue
            name = d["Kernel Name"].split("(")[0].replace("tpcb::<unnamed>::", "")
            agg[name][0] += 1
            agg[name][1] += float(d["Metric Value"]) / 1e3
    tot = sum(v[1] for v in agg.values())
    for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{k[:70]:70s} n={n:5d} total {t:10.1f} us  avg {t / n:8.2f} us  share {100 * t / tot:5.1f}%")


def full(path, ids=None):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        if ids and d["ID"] not in ids:
            continue
        print(f"[{d['ID']}] {d['Kernel Name'][:100]}")
        for k in KEYS:
            if k in d:
                print(f"    {k:70s} {d[k]:>16s} {units[hdr.index(k)]}")


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2])
    else:
        full(sys.argv[2], sys.argv[3:] or None)
