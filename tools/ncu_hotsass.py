"""Top SASS instructions by warp-stall samples of one kernel in an ncu report:
    python tools/ncu_hotsass.py REP KERNEL_REGEX [N]"""
import csv
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", "regex:" + kre,
                      "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
si = hdr.index("Warp Stall Sampling (All Samples)")
stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
body = [r for r in rows[2:] if len(r) > si and r[si].isdigit()]
tot = sum(int(r[si]) for r in body) or 1
print("total samples", tot)
for r in sorted(body, key=lambda r: -int(r[si]))[:n]:
    top = sorted(((int(r[i]) if r[i].isdigit() else 0, hdr[i][6:]) for i in stall_cols), reverse=True)[:3]
    print(f"{100 * int(r[si]) / tot:5.1f}%  {r[1].strip()[:58]:58s} " + " ".join(f"{k}={v}" for v, k in top if v))
