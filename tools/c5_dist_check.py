"""Config 5 end to end on G GPUs (torchrun): 100 M samples, 100 epochs, 8192 workers built by
DistributedPlan (epoch-sharded shuffle with the fused peer-memory exchange, worker-sharded
build, holder-offset merge), then checked against the reference's own functions on a worker
subset (8 workers per rank, both edges of every rank's range): streams, class lists, and the
subset-restricted holder CSR (every subset holder record in sample / worker order).
    python -m torch.distributed.run --nproc-per-node 4 --master-addr 127.0.0.1 tools/c5_dist_check.py"""
import os
import sys
import time

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from paper_2101_08734_b200 import clairplan as cp  # noqa: E402
from paper_2101_08734_b200.distributed import DistributedPlan  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
    dist.init_process_group("nccl", device_id=torch.device("cuda", torch.cuda.current_device()))
    F, N, b, E = 100_000_000, 8192, 32, 100
    caps = [120_000.0, 900_000.0]
    sizes = cp.generate_sizes(F, 0.1077, 0.1, None, 1)
    t0 = time.time()
    dp = DistributedPlan(42, F, cp.PartitionSpec(N, b * N, E, True), caps, sizes).build()
    torch.cuda.synchronize()
    st = dp.plan.stats()
    wb, we = dp.wrange
    rng = np.random.default_rng(rank)
    mine = sorted({wb, wb + 1, we - 2, we - 1} | {int(x) for x in rng.integers(wb, we, 4)})
    streams = {w: dp.plan.stream(w) for w in mine}
    cls = dp.plan.class_lists()
    lists = {w: cls[w - wb] for w in mine}
    offs, hold = dp.plan.holders()
    keep = np.isin(hold[:, 0], np.array(mine, np.uint32))
    owner = np.repeat(np.arange(F, dtype=np.int64), np.diff(offs.astype(np.int64)))
    sub = (owner[keep], hold[keep])
    print(f"rank {rank}: workers [{wb}, {we}) built in {time.time() - t0:.1f} s, A {st['accesses']}, "
          f"D {st['pairs']}, path {st['path']}, p2p {dp.p2p}", flush=True)
    dp.close()
    parts = [None] * world
    dist.all_gather_object(parts, (mine, streams, lists, sub))
    ok = True
    if rank == 0:
        from _oracle import Ref
        subset = np.array(sorted(w for p in parts for w in p[0]), np.uint32)
        t1 = time.time()
        ref = Ref().plan_subset_lowmem(42, F, N, b * N, E, True, caps,
                                       cp.generate_sizes(F, 0.1077, 0.1, None, 1), subset,
                                       os.cpu_count() or 8)
        print(f"reference subset ({len(subset)} workers) {time.time() - t1:.1f} s", flush=True)
        for mine, streams, lists, _ in parts:
            for w in mine:
                ok &= bool(np.array_equal(streams[w], ref.streams[w]))
                ok &= all(np.array_equal(lists[w][j], ref.class_lists[w][j]) for j in range(2))
        # subset-restricted CSR: records in (sample, worker) order, shards in rank order
        k_all = np.concatenate([p[3][0] for p in parts])
        h_all = np.concatenate([p[3][1] for p in parts])
        order = np.lexsort((h_all[:, 0], k_all))
        roffs = ref.holder_offsets.astype(np.int64)
        rk = np.repeat(np.arange(F, dtype=np.int64), np.diff(roffs))
        ok &= bool(np.array_equal(k_all[order], rk) and np.array_equal(h_all[order], ref.holders))
        print(f"c5_dist_check world {world}: {len(subset)} subset workers, "
              f"{len(ref.holders)} holder records: {'OK' if ok else 'FAILED'}", flush=True)
    t = torch.tensor([1 if ok else 0], device="cuda")
    dist.broadcast(t, 0)
    dist.destroy_process_group()
    sys.exit(0 if int(t) == 1 else 1)


if __name__ == "__main__":
    main()
