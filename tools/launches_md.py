"""ncu launch-list CSV -> markdown summary (per-kernel ms, share, DRAM MB) for profiles/:
    python tools/launches_md.py launches.csv "title" [plans]"""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
title = sys.argv[2] if len(sys.argv) > 2 else sys.argv[1]
plans = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
hdr = rows[0]
ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
agg = collections.defaultdict(lambda: collections.defaultdict(float))
cnt = collections.Counter()
for r in rows[1:]:
    k = r[ki].split("(")[0].replace("void ", "")
    agg[k][r[mi]] += float(r[vi].replace(",", ""))
    if r[mi] == "gpu__time_duration.sum":
        cnt[k] += 1
tot = sum(m["gpu__time_duration.sum"] for m in agg.values()) / 1e6 / plans
rd = sum(m.get("dram__bytes_read.sum", 0) for m in agg.values()) / 1e6 / plans
wr = sum(m.get("dram__bytes_write.sum", 0) for m in agg.values()) / 1e6 / plans
print(f"# {title}\n")
print("Per-launch device times from `ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,"
      "dram__bytes_write.sum --clock-control none` (cold-cache, serialised: compare shares, "
      "not absolutes).\n")
print("| kernel | launches | total ms | share | DRAM read MB | DRAM write MB |")
print("|---|---:|---:|---:|---:|---:|")
for k, m in sorted(agg.items(), key=lambda x: -x[1]["gpu__time_duration.sum"]):
    ms = m["gpu__time_duration.sum"] / 1e6 / plans
    if ms < 0.001:
        continue
    print(f"| `{k}` | {cnt[k] / plans:g} | {ms:.3f} | {100 * ms / tot:.1f}% | "
          f"{m.get('dram__bytes_read.sum', 0) / 1e6 / plans:.1f} | "
          f"{m.get('dram__bytes_write.sum', 0) / 1e6 / plans:.1f} |")
print(f"\nTotal clairplan kernels: {tot:.3f} ms, DRAM {rd / 1e3:.2f} GB read + {wr / 1e3:.2f} GB "
      f"written = {(rd + wr) / 1e3:.2f} GB per plan.")
