#!/usr/bin/env python
"""Print the key per-kernel metrics of an ncu report (ncu -i REP --page details --csv)."""
import csv
import subprocess
import sys

WANT = ["Duration", "DRAM Throughput", "Memory Throughput", "L2 Hit Rate", "L1/TEX Hit Rate",
        "Achieved Occupancy", "Registers Per Thread", "Compute (SM) Throughput",
        "Issued Warp Per Scheduler", "Eligible Warps Per Scheduler",
        "Warp Cycles Per Issued Instruction", "Dynamic Shared Memory Per Block"]


def main(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True,
                         text=True).stdout
    lines = out.splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    r = list(csv.reader(lines[start:]))
    hdr = r[0]
    ki, mi, vi, ui = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value",
                                             "Metric Unit"))
    idi = hdr.index("ID")
    cur = None
    for row in r[1:]:
        key = (row[idi], row[ki].split("(")[0])
        if key != cur:
            print("==", key[1], "(id", key[0] + ")")
            cur = key
        if row[mi] in WANT:
            print(f"    {row[mi]:38s} {row[vi]} {row[ui]}")


if __name__ == "__main__":
    main(sys.argv[1])
