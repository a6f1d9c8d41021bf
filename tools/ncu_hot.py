#!/usr/bin/env python
"""Top SASS instructions by warp-stall samples for one kernel of an ncu report."""
import csv
import subprocess
import sys


def main(rep, kern, n=30):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name",
                          f"regex:{kern}"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = next(r for r in rows if r and r[0] == "Address")
    data = [r for r in rows[rows.index(hdr) + 1:] if r and r[0] != 'Address' and r[0].startswith('0x')]
    si = hdr.index("Warp Stall Sampling (All Samples)")
    ii = hdr.index("Instructions Executed")
    tot = sum(float((r[si] or '0').replace(',', '')) for r in data if len(r) > si) or 1
    print(f"{kern}: {len(data)} SASS lines, {tot:.0f} stall samples")
    for idx, r in sorted(enumerate(data), key=lambda x: -float((x[1][si] or '0').replace(',', '')))[:n]:
        print(f"{100 * float(r[si].replace(',', '')) / tot:5.1f}%  #{idx:5d} exec={r[ii]:>9s}  {r[1][:100]}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 30)
