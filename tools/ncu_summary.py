"""Summarise an ncu report (or a launch-list CSV) into the small text/JSON files
committed under profiles/.

    python tools/ncu_summary.py report.ncu-rep  > profiles/<name>.txt
    python tools/ncu_summary.py --launches launches.csv > profiles/<name>_launches.txt
    python tools/ncu_summary.py --traffic report.ncu-rep --key cfg2_w4a4_m1 [--json profiles/ncu_traffic.json]
"""
from __future__ import annotations

import argparse
import collections
import csv
import io
import json
import subprocess
import sys

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
]


def raw_rows(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[2:], rows[1]


_BYTE_SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def to_bytes(value, unit):
    """ncu picks a unit per metric per report (row 2 of the raw CSV); normalise to bytes."""
    return float(value.replace(",", "")) * _BYTE_SCALE[unit.strip()]


def summary(path):
    h, rows, units = raw_rows(path)
    for r in rows:
        name = r[h.index("Kernel Name")] if "Kernel Name" in h else "?"
        print(f"kernel: {name}")
        for m in METRICS:
            if m in h:
                print(f"  {m:70s} {r[h.index(m)]} {units[h.index(m)]}")
        stalls = [(c, r[i]) for i, c in enumerate(h) if "pcsamp_warps_issue_stalled" in c and not c.endswith("not_issued")]
        stalls = sorted(stalls, key=lambda x: -float(x[1] or 0))[:6]
        if stalls:
            print("  top stall reasons (samples): " + ", ".join(f"{c.split('stalled_')[-1]}={v}" for c, v in stalls))


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hdr]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = collections.defaultdict(list)
    for r in rows[hdr + 1:]:
        if len(r) > vi:
            agg[r[ki][:90]].append(float(r[vi].replace(",", "")))
    tot = sum(sum(v) for v in agg.values())
    print(f"{'n':>5} {'mean us':>9} {'share':>6}  kernel")
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        print(f"{len(v):5d} {sum(v) / len(v) / 1000:9.3f} {sum(v) / tot * 100:5.1f}%  {k}")


def traffic(path, key, json_path):
    h, rows, units = raw_rows(path)
    r = rows[0]
    b = sum(to_bytes(r[h.index(m)], units[h.index(m)]) for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
    rec = {"dram_bytes_per_launch": int(b), "source": path,
           "units": [units[h.index(m)] for m in ("dram__bytes_read.sum", "dram__bytes_write.sum")]}
    data = {}
    if json_path:
        try:
            data = json.load(open(json_path))
        except FileNotFoundError:
            data = {}
        data[key] = rec
        json.dump(data, open(json_path, "w"), indent=1)
    print(json.dumps({key: rec}))


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("path")
    ap.add_argument("--launches", action="store_true")
    ap.add_argument("--traffic", action="store_true")
    ap.add_argument("--key", default="cfg2_w4a4_m1")
    ap.add_argument("--json", default=None)
    a = ap.parse_args()
    if a.launches:
        launches(a.path)
    elif a.traffic:
        traffic(a.path, a.key, a.json)
    else:
        summary(a.path)
    sys.exit(0)
