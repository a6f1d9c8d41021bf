"""Per-kernel totals of an ncu --csv --metrics launch list: python tools/agg_ncu.py file.csv [div]"""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
div = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
agg = collections.defaultdict(lambda: collections.defaultdict(float))
cnt = collections.Counter()
for r in rows[1:]:
    k = r[ki].split("(")[0]
    agg[k][r[mi]] += float(r[vi].replace(",", ""))
    if r[mi] == "gpu__time_duration.sum":
        cnt[k] += 1
for k, m in sorted(agg.items(), key=lambda x: -x[1]["gpu__time_duration.sum"]):
    print(f"{k:40s} n={cnt[k] / div:5.1f} ms={m['gpu__time_duration.sum'] / 1e6 / div:8.3f} "
          + " ".join(f"{n.split('__')[1].split('.')[0]}={v / div / 1e6:9.1f}M" for n, v in m.items()
                     if n != "gpu__time_duration.sum"))
