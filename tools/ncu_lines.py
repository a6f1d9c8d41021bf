#!/usr/bin/env python
"""Per CUDA source line: warp-stall samples and warp instructions executed, for one kernel
of an ncu report (needs -lineinfo + --import-source on).

    python tools/ncu_lines.py REP KERNEL_REGEX [top]
"""
import collections
import csv
import subprocess
import sys


def main(rep, kern, top=40):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                          "sass,cuda", "-k", f"regex:{kern}"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    stall = collections.Counter()
    inst = collections.Counter()
    src = {}
    fname = ""
    hdr = None
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].rsplit("/", 1)[-1]
            hdr = None
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) < len(hdr) or not r[0].isdigit():
            continue
        key = (fname, int(r[0]))
        src[key] = r[1].strip()[:90]
        try:
            stall[key] += float((r[4] or "0").replace(",", ""))
            inst[key] += float((r[7] or "0").replace(",", ""))
        except ValueError:
            pass
    ts = sum(stall.values()) or 1
    ti = sum(inst.values()) or 1
    print(f"{kern}: {ts:.0f} stall samples, {ti:.3e} warp instructions")
    for key, v in stall.most_common(int(top)):
        print(f"{100 * v / ts:5.1f}% st {100 * inst[key] / ti:5.1f}% in  {key[0]}:{key[1]:<5d} {src[key]}")


if __name__ == "__main__":
    main(*sys.argv[1:])
