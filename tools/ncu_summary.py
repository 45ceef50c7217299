"""Summarise ncu outputs into text for profiles/ (run in the build container).

    python tools/ncu_summary.py launches <launches.csv>      # per-kernel device times
    python tools/ncu_summary.py report <file.ncu-rep> [regex]  # key metrics per kernel
"""
import csv
import io
import re
import subprocess
import sys
from collections import defaultdict

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__cycles_elapsed.avg.per_second",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr, per = None, defaultdict(list)
    order = []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                name = re.sub(r"\(.*", "", d["Kernel Name"]).strip()
                if name not in per:
                    order.append(name)
                per[name].append(float(d["Metric Value"].replace(",", "")))
    tot = sum(sum(v) for v in per.values())
    print(f"{'kernel':70s} {'launches':>8s} {'avg_us':>10s} {'share':>7s}")
    for n in order:
        v = per[n]
        print(f"{n[:70]:70s} {len(v):8d} {sum(v)/len(v)/1e3:10.1f} {sum(v)/tot*100:6.1f}%")


def report(path, regex=None):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        name = d.get("Kernel Name", "")
        if regex and not re.search(regex, name):
            continue
        print(f"== {name[:110]}")
        for k in KEYS:
            if k in d:
                print(f"   {k:75s} {d[k]:>16s} {units[hdr.index(k)]}")


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2])
    else:
        report(sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else None)
