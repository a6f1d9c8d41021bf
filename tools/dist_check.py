"""Multi-GPU parity check (run with torchrun, one rank per GPU):
    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 tools/dist_check.py
Every rank builds its shard through DistributedPlan (epoch-range streams + NCCL all-to-all +
worker-range build + holder-offset merge; and the older permutation all-gather mode) and
compares it with a single-GPU plan of all workers built locally."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2101_08734_b200 import clairplan as cp  # noqa: E402
from paper_2101_08734_b200.distributed import DistributedPlan  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
    dist.init_process_group("nccl", device_id=torch.device("cuda", torch.cuda.current_device()))
    ok = True
    cases = [(1_281_167, 256, 32, 9, True, "streams", None), (262_144, 64, 16, 10, True, "streams", None),
             (20_000, 7, 5, 13, True, "streams", None), (20_011, 9, 3, 7, False, "streams", None),
             (30_000, 5, 7, 3, False, "streams", None), (40_000, 16, 8, 12, True, "streams", [1e9, 1e9]),
             (1_281_167, 256, 32, 9, True, "dense", None), (20_011, 9, 3, 7, False, "dense", None),
             (1_281_167, 256, 32, 9, True, "sparse", None), (20_011, 9, 3, 7, False, "sparse", None),
             (262_144, 64, 16, 10, True, "sparse", [50.0, 1e9]), (30_000, 5, 7, 3, False, "sparse", None),
             (1_281_167, 256, 32, 9, True, "perms", None), (20_000, 7, 5, 13, True, "perms", None),
             (20_011, 9, 3, 7, False, "pipelined", None), (1_281_167, 256, 32, 9, True, "pipelined", None),
             (1_281_167, 256, 32, 9, True, "p2p", None), (20_011, 9, 3, 7, False, "p2p", None),
             (262_144, 64, 16, 10, True, "p2p", [50.0, 1e9]), (20_000, 7, 5, 13, True, "p2p2", None),
             (1_281_167, 256, 32, 9, True, "p2p2", None)]
    for (F, N, b, E, dl, mode, caps) in cases:
        sizes = cp.generate_sizes(F, 0.1077, 0.1, None, 1)
        part = cp.PartitionSpec(N, b * N, E, dl)
        caps = caps or [120.0 * F / 1e4, 900.0 * F / 1e4]
        if mode in ("dense", "sparse"):  # streams mode, forced sample-major pass flavour
            os.environ["CLAIRPLAN_DENSE"] = "1" if mode == "dense" else "0"
        dmode = "perms" if mode == "perms" else "p2p" if mode.startswith("p2p") else "streams"
        dp = DistributedPlan(42, F, part, caps, sizes, mode=dmode,
                             pipeline=(mode == "pipelined")).build()
        if mode == "p2p2":  # second build: the other receive buffer
            dp.build()
        if mode.startswith("p2p") and not dp.p2p:
            print(f"rank {rank}: p2p mode not taken", flush=True)
            ok = False
        os.environ.pop("CLAIRPLAN_DENSE", None)
        full = cp.Plan(42, F, part, caps, sizes, device=torch.cuda.current_device()).build()
        wb, we = dp.wrange
        st_full = full.streams_flat()
        st_mine = dp.plan.streams_flat()
        offs_full, hold_full = full.holders()
        # streams of my workers
        lo = cp.lib().clairplan_stream_offset(full._h, wb)
        hi = cp.lib().clairplan_stream_offset(full._h, we)
        ok &= np.array_equal(st_full[lo:hi], st_mine)
        # class lists of my workers
        cl_full, cl_mine = full.class_lists()[wb:we], dp.plan.class_lists()
        ok &= all(np.array_equal(x, y) for a, c in zip(cl_full, cl_mine) for x, y in zip(a, c))
        # holder CSR: global offsets and my records at their global positions
        ok &= np.array_equal(dp.global_offsets.cpu().numpy(), offs_full.astype(np.int64))
        offs_mine, hold_mine = dp.plan.holders()
        starts = dp.rank_starts.cpu().numpy()
        cnt = np.diff(offs_mine.astype(np.int64))
        H = int(cnt.sum())
        if starts.shape != cnt.shape or hold_mine.shape[0] != H:
            print(f"rank {rank}: shape mismatch starts {starts.shape} cnt {cnt.shape} "
                  f"holders {hold_mine.shape} offs {offs_mine.shape}", flush=True)
            ok = False
        else:
            within = np.arange(H, dtype=np.int64) - np.repeat(offs_mine[:-1].astype(np.int64), cnt)
            pos = np.repeat(starts.astype(np.int64), cnt) + within
            ok &= bool(np.array_equal(hold_full[pos], hold_mine))
        print(f"rank {rank} F={F} N={N} E={E} dl={dl} mode={mode} ok={ok}", flush=True)
        dp.close()
        full.close()
    t = torch.tensor([1 if ok else 0], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MIN)
    if rank == 0:
        print("dist_check", "OK" if int(t) == 1 else "FAILED", "world", world)
    dist.destroy_process_group()
    sys.exit(0 if int(t) == 1 else 1)


if __name__ == "__main__":
    main()
