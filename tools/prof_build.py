"""Builds one benchmark configuration `reps` times (for ncu launch lists / captures):
    python tools/prof_build.py [config] [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2101_08734_b200 import clairplan as cp  # noqa: E402


def main():
    c = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    cfg = bench.CONFIGS[c]
    mu, sd, tot = cfg["sizes"]
    sizes = cp.generate_sizes(cfg["F"], mu, sd, tot, 1)
    part = cp.PartitionSpec(cfg["N"], cfg["b"] * cfg["N"], cfg["E"], True)
    plan = cp.Plan(bench.SEED, cfg["F"], part, list(bench.CAPS), sizes, device=0)
    for _ in range(reps):
        plan.build()
    torch.cuda.synchronize()
    print("built", reps)


if __name__ == "__main__":
    main()
