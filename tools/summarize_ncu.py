#!/usr/bin/env python
"""Summarise an ncu --csv launch list (gpu__time_duration + dram bytes per kernel).

    python tools/summarize_ncu.py gpurun_out/launches.csv profiles/r01_launches.md \
        [--traffic profiles/traffic_latest.json --workload imagenet1k-e90-n256]

Writes a markdown table (per kernel: launches, total/mean time, share, DRAM read/write) and,
optionally, the per-plan DRAM traffic of the clairplan kernels for bench.py's roofline.
"""
import argparse
import collections
import csv
import json


def load(path):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    return data


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("out_md")
    ap.add_argument("--traffic")
    ap.add_argument("--workload", default="")
    ap.add_argument("--title", default="")
    ap.add_argument("--reps", type=float, default=1.0, help="plans in the launch list")
    a = ap.parse_args()
    data = load(a.csv)
    agg = collections.OrderedDict()
    for d in data:
        name = d["Kernel Name"].split("(")[0].replace("void ", "")
        m, v = d["Metric Name"], float(d["Metric Value"].replace(",", ""))
        unit = d["Metric Unit"]
        x = agg.setdefault(name, {"n": 0, "ns": 0.0, "rd": 0.0, "wr": 0.0})
        if m == "gpu__time_duration.sum":
            x["ns"] += v * (1e3 if unit == "us" else 1e6 if unit == "ms" else 1.0)
            x["n"] += 1
        elif m == "dram__bytes_read.sum":
            x["rd"] += v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
        elif m == "dram__bytes_write.sum":
            x["wr"] += v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
    # ncu may or may not print the clairplan:: namespace; drop torch's own kernels
    ours = {k: v for k, v in agg.items() if "at::" not in k and "native::" not in k}
    for v in ours.values():
        for f in ("n", "ns", "rd", "wr"):
            v[f] /= a.reps
    tot = sum(v["ns"] for v in ours.values())
    lines = [f"# {a.title or 'ncu launch list'}", "",
             "Per-launch device times from `ncu --metrics gpu__time_duration.sum,"
             "dram__bytes_read.sum,dram__bytes_write.sum --clock-control none` (cold-cache, "
             "serialised: compare shares, not absolutes).", "",
             "| kernel | launches | total ms | share | DRAM read MB | DRAM write MB |",
             "|---|---:|---:|---:|---:|---:|"]
    for k, v in sorted(ours.items(), key=lambda kv: -kv[1]["ns"]):
        lines.append(f"| `{k.replace('clairplan::', '')}` | {v['n']:g} | {v['ns'] / 1e6:.3f} | "
                     f"{100 * v['ns'] / tot:.1f}% | {v['rd'] / 1e6:.1f} | {v['wr'] / 1e6:.1f} |")
    rd = sum(v["rd"] for v in ours.values())
    wr = sum(v["wr"] for v in ours.values())
    lines += ["", f"Total clairplan kernels: {tot / 1e6:.3f} ms, DRAM {rd / 1e9:.3f} GB read + "
              f"{wr / 1e9:.3f} GB written = {(rd + wr) / 1e9:.3f} GB per plan."]
    open(a.out_md, "w").write("\n".join(lines) + "\n")
    if a.traffic:
        json.dump({"workload": a.workload, "dram_bytes_per_plan": rd + wr,
                   "kernel_ms_serialised": tot / 1e6, "source": a.csv}, open(a.traffic, "w"),
                  indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
