#!/usr/bin/env python
"""Per-source-line instruction and stall shares of one kernel in an ncu report
(compile with -lineinfo, capture with --import-source on).

  python scripts/ncu_lines.py REPORT.ncu-rep [top]

Prints the top lines by executed warp-instructions with their share of the
kernel's instructions and of its warp-stall samples."""
import collections
import csv
import io
import subprocess
import sys


def main(rep, top=60):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         check=True, capture_output=True, text=True).stdout
    cur_file, cur_line = None, None
    inst, stall, src = collections.Counter(), collections.Counter(), {}
    head = None
    for r in csv.reader(io.StringIO(txt)):
        if len(r) == 2 and r[0] == "File Path":
            cur_file = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            head = r
            continue
        if head is None or len(r) < 8:
            continue
        if r[0] != "":
            cur_line = (cur_file, int(r[0]))
            src[cur_line] = r[1].strip()[:100]
            continue
        try:
            ie = int(r[head.index("Instructions Executed")])
            st = int(r[head.index("Warp Stall Sampling (All Samples)")])
        except (ValueError, IndexError):
            continue
        inst[cur_line] += ie
        stall[cur_line] += st
    ti, ts = sum(inst.values()) or 1, sum(stall.values()) or 1
    print(f"total warp instructions {ti}, stall samples {ts}")
    for k, v in sorted(inst.items(), key=lambda x: -x[1])[:top]:
        print(f"{k[0]}:{k[1]:5d} {100 * v / ti:5.1f}% inst {100 * stall[k] / ts:5.1f}% stall  {src.get(k, '')}")
    print("-- top by stall samples")
    for k, v in sorted(stall.items(), key=lambda x: -x[1])[:25]:
        print(f"{k[0]}:{k[1]:5d} {100 * inst[k] / ti:5.1f}% inst {100 * v / ts:5.1f}% stall  {src.get(k, '')}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 60)
