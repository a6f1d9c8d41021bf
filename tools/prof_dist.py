"""Builds one benchmark configuration through DistributedPlan (streams mode) `reps` times on
the ranks of a torchrun launch (also world size 1), for ncu launch lists / stage timing:
    python -m torch.distributed.run --nproc-per-node G tools/prof_dist.py [config] [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import bench  # noqa: E402
from paper_2101_08734_b200 import clairplan as cp  # noqa: E402
from paper_2101_08734_b200.distributed import DistributedPlan  # noqa: E402


def main():
    c = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg = bench.CONFIGS[c]
    mu, sd, tot = cfg["sizes"]
    sizes = cp.generate_sizes(cfg["F"], mu, sd, tot, 1)
    part = cp.PartitionSpec(cfg["N"], cfg["b"] * cfg["N"], cfg["E"], True)
    dp = DistributedPlan(bench.SEED, cfg["F"], part, list(bench.CAPS), sizes)
    for _ in range(reps):
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record()
        dp.build()
        ev1.record()
        ev1.synchronize()
        if dist.get_rank() == 0:
            print("build ms", round(ev0.elapsed_time(ev1), 3), dp.timings, flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
