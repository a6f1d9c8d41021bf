"""Builds one benchmark configuration `reps` times (for ncu launch lists / captures):
    python tools/prof_build.py [config] [reps] [shards]
shards > 1: the handle plans only the first 1/shards of the workers (one rank's worker range
of a sharded build; the permutations still cover every epoch)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2101_08734_b200 import clairplan as cp  # noqa: E402


def main():
    c = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    shards = int(sys.argv[3]) if len(sys.argv) > 3 else 1
    cfg = bench.CONFIGS[c]
    mu, sd, tot = cfg["sizes"]
    sizes = cp.generate_sizes(cfg["F"], mu, sd, tot, 1)
    part = cp.PartitionSpec(cfg["N"], cfg["b"] * cfg["N"], cfg["E"], True)
    plan = cp.Plan(bench.SEED, cfg["F"], part, list(bench.CAPS), sizes, device=0,
                   worker_range=(0, cfg["N"] // shards))
    for _ in range(reps):
        plan.build()
        st = plan.stats()
    torch.cuda.synchronize()
    print("built", reps, "device_ms", round(st["device_ms"], 3), st["path"])


if __name__ == "__main__":
    main()
