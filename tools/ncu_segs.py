#!/usr/bin/env python
"""Straight-line SASS segments of one kernel ranked by executed instructions:
    python tools/ncu_segs.py REP KERNEL_REGEX [N]"""
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = next(r for r in rows if r and r[0] == "Address")
data = [r for r in rows[rows.index(hdr) + 1:] if r and r[0].startswith("0x")]
seen, uniq = set(), []
for r in data:  # the page may list the function twice
    if r[0] in seen:
        break
    seen.add(r[0])
    uniq.append(r)
ii, si = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
tot = sum(float(r[ii] or 0) for r in uniq)
print(f"{kern}: {len(uniq)} SASS lines, {tot:.0f} warp instructions")
segs, cur = [], None
for k, r in enumerate(uniq):
    v, s = int(float(r[ii] or 0)), int(float(r[si] or 0))
    if cur and cur[1] == v:
        cur[2] += 1
        cur[3] += s
    else:
        cur = [k, v, 1, s, r[1][:70]]
        segs.append(cur)
for sg in sorted(segs, key=lambda x: -x[1] * x[2])[:n]:
    print(f"#{sg[0]:5d} exec={sg[1]:>9d} x{sg[2]:3d} = {100 * sg[1] * sg[2] / tot:5.1f}%  stall={sg[3]:6d}  {sg[4]}")
