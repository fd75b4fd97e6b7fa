#!/usr/bin/env python
"""Summarise `ncu --set full` captures into profiles/union_ncu_summary.json.

  python scripts/ncu_summary.py KEY REPORT.ncu-rep [KEY REPORT ...] [--kernel REGEX]

Each KEY (e.g. c3_p10) gets the per-launch figures bench.py's `roofline` uses:
issued warp-instructions, DRAM bytes, duration, SM clock, pipe utilisations,
cache hit rates and stall reasons.  The instruction and DRAM counts are
per-launch constants of a kernel on a given graph, so bench.py divides them by
the LIVE launch time it measures with CUDA events (ncu's own times are
serialised and cold-cache).
"""
from __future__ import annotations

import csv
import io
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "profiles", "union_ncu_summary.json")

METRICS = {
    "duration_ms": "gpu__time_duration.sum",
    "sm_clock_ghz": "sm__cycles_elapsed.avg.per_second",
    "warp_instructions_issued": "smsp__inst_issued.sum",
    "issue_active_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "alu_pipe_pct": "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "fma_pipe_pct": "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "lsu_pipe_pct": "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "l1_throughput_pct": "l1tex__throughput.avg.pct_of_peak_sustained_active",
    "l1_data_pipe_pct": "l1tex__data_pipe_lsu_wavefronts.sum.pct_of_peak_sustained_elapsed",
    "l1_hit_rate_pct": "l1tex__t_sector_hit_rate.pct",
    "l2_hit_rate_pct": "lts__t_sector_hit_rate.pct",
    "dram_bytes_read": "dram__bytes_read.sum",
    "dram_bytes_write": "dram__bytes_write.sum",
    "registers_per_thread": "launch__registers_per_thread",
    "grid_size": "launch__grid_size",
    "achieved_warps_per_sm": "sm__warps_active.avg.per_cycle_active",
}
UNIT_SCALE = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "Tbyte": 1e12, "usecond": 1e-3, "us": 1e-3,
              "ms": 1.0, "msecond": 1.0, "ns": 1e-6, "nsecond": 1e-6, "s": 1e3, "second": 1e3}


def read_raw(rep: str, kernel: str | None):
    cmd = ["ncu", "-i", rep, "--page", "raw", "--csv"]
    if kernel:
        cmd += ["-k", f"regex:{kernel}"]
    txt = subprocess.run(cmd, check=True, capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    head, units, data = rows[0], rows[1], rows[2:]
    return head, units, data


def value(head, units, row, name):
    i = head.index(name)
    s = row[i].replace(",", "")
    if s in ("", "n/a"):
        return None
    v = float(s)
    u = units[i]
    if name.startswith("dram__bytes"):
        v *= UNIT_SCALE.get(u, 1.0)
    elif name == "gpu__time_duration.sum":
        v *= UNIT_SCALE.get(u, 1.0)
    return v


def summarise(rep: str, kernel: str | None) -> dict:
    head, units, data = read_raw(rep, kernel)
    if not data:
        raise SystemExit(f"{rep}: no kernel matched")
    row = data[0]
    out = {"kernel": row[head.index("Kernel Name")]}
    for key, name in METRICS.items():
        if name in head:
            out[key] = value(head, units, row, name)
    out["dram_bytes_per_launch"] = (out.get("dram_bytes_read") or 0) + (out.get("dram_bytes_write") or 0)
    stalls = {}
    for i, h in enumerate(head):
        m = re.match(r"smsp__average_warps_issue_stalled_(\w+)_per_issue_active\.ratio", h)
        if m and row[i] not in ("", "n/a"):
            stalls[m.group(1)] = float(row[i])
    out["stalls_per_issue"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1])[:6])
    out["source"] = os.path.basename(rep).replace(".ncu-rep", "") + " (ncu --set full --clock-control none)"
    return out


def main(argv):
    global OUT
    if "--out" in argv:
        i = argv.index("--out")
        OUT = argv[i + 1]
        argv = argv[:i] + argv[i + 2:]
    kernel = None
    if "--kernel" in argv:
        i = argv.index("--kernel")
        kernel = argv[i + 1]
        argv = argv[:i] + argv[i + 2:]
    pairs = list(zip(argv[0::2], argv[1::2]))
    db = json.load(open(OUT)) if os.path.exists(OUT) else {}
    for key, rep in pairs:
        db[key] = summarise(rep, kernel)
        print(key, json.dumps(db[key], indent=1))
    with open(OUT, "w") as f:
        json.dump(db, f, indent=1)
        f.write("\n")


if __name__ == "__main__":
    main(sys.argv[1:])
