"""Config 5 (100 M samples, 100 epochs, 8192 workers) through the sharded build, checked
against the reference for a worker subset (run with torchrun, one rank per GPU):
    python -m torch.distributed.run --nproc-per-node G tools/c5_check.py [F] [E] [N]
Every rank builds its shard (epoch-range streams + all-to-all + worker-range build + holder
merge); rank 0 runs the reference's own functions for the subset (epoch by epoch, so the
100 permutations never sit in host memory together) and every rank compares its subset
workers' streams and class lists, and its records of the subset-restricted holder CSR."""
import ctypes as C
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


class _Dev:
    def __init__(self, ptr, n, typestr):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr, "data": (ptr, False),
                                         "version": 3}


def dev_tensor(ptr, n, typestr):
    """A torch view of library device memory (no copy)."""
    return torch.as_tensor(_Dev(ptr, n, typestr), device="cuda")


def main():
    F = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000_000
    E = int(sys.argv[2]) if len(sys.argv) > 2 else 100
    N = int(sys.argv[3]) if len(sys.argv) > 3 else 8192
    b = 32
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
    dist.init_process_group("nccl", device_id=torch.device("cuda", torch.cuda.current_device()))
    caps = [120_000.0, 900_000.0]
    sizes = cp.generate_sizes(F, 0.1077, 0.1, None, 1)
    part = cp.PartitionSpec(N, b * N, E, True)
    t0 = time.time()
    dp = DistributedPlan(42, F, part, caps, sizes).build()
    torch.cuda.synchronize()
    t1 = time.time()
    st = dp.stats()
    wb, we = dp.wrange
    # subset: both ends of every rank's range plus fixed pseudo-random workers
    rng = np.random.default_rng(5)
    subset = sorted(set([0, 1, N - 2, N - 1] + [int(r * N // world) for r in range(world)] +
                        [int((r + 1) * N // world) - 1 for r in range(world)] +
                        [int(x) for x in rng.integers(0, N, 16)]))
    subset = np.array(subset, np.uint32)
    print(f"rank {rank}: build {t1 - t0:.1f} s, A {st['accesses']}, D {st['pairs']}, "
          f"path {st['path']}, timings {dp.timings}", flush=True)
    ok = True
    if rank == 0:
        from _oracle import Ref
        t2 = time.time()
        ref = Ref().plan_subset_lowmem(42, F, N, b * N, E, True, caps, sizes, subset,
                                       os.cpu_count() or 8)
        print(f"reference subset plan {time.time() - t2:.1f} s", flush=True)
        payload = [ref]
    else:
        payload = [None]
    # every rank compares what it owns; the reference's subset data is broadcast (per-sample
    # subset holder counts as u8, the subset's streams / class lists / holder records)
    ref = payload[0]
    mine = [int(w) for w in subset if wb <= w < we]
    obj = [None]
    if rank == 0:
        obj = [{"streams": {int(w): ref.streams[w] for w in subset},
                "class_lists": {int(w): ref.class_lists[w] for w in subset},
                "counts": np.diff(ref.holder_offsets.astype(np.int64)).astype(np.uint8),
                "holders": ref.holders}]
        del ref
    dist.broadcast_object_list(obj, src=0)
    R = obj[0]
    for w in mine:
        ok &= bool(np.array_equal(dp.plan.stream(w), R["streams"][w]))
    # class lists and holders of the subset from device views (the shard's full host export
    # would be tens of GB)
    L = cp.lib()
    J = len(caps)
    nloc = we - wb
    off = np.zeros(nloc * J, np.uint64)
    ln = np.zeros(nloc * J, np.uint64)
    cp._check(L.clairplan_class_list_bounds(dp.plan._h, off.ctypes.data_as(cp.u64p),
                                            ln.ctypes.data_as(cp.u64p)))
    ent = cp.u32p()
    cp._check(L.clairplan_device_class_lists(dp.plan._h, C.byref(ent)))
    ent_ptr = C.cast(ent, C.c_void_p).value
    for w in mine:
        for j in range(J):
            o, n = int(off[(w - wb) * J + j]), int(ln[(w - wb) * J + j])
            got = dev_tensor(ent_ptr + 4 * o, n, "<i4").cpu().numpy().view(np.uint32) if n else \
                np.zeros(0, np.uint32)
            ok &= bool(np.array_equal(got, R["class_lists"][w][j]))
    po, ph, H = dp.plan.device_holders()
    offs = dev_tensor(po, F + 1, "<i8")
    h3 = dev_tensor(ph, 3 * H, "<i4").view(-1, 3)
    sub_t = torch.tensor(subset.astype(np.int64), device="cuda").to(torch.int32)
    mask = torch.isin(h3[:, 0], sub_t)
    idx = mask.nonzero().squeeze(1)
    mk = (torch.searchsorted(offs, idx.to(torch.int64), right=True) - 1).cpu().numpy()
    mine_h = h3[idx].cpu().numpy().view(np.uint32)
    roffs = np.zeros(F + 1, np.int64)
    roffs[1:] = np.cumsum(R["counts"].astype(np.int64))
    rh = R["holders"]
    rowner = np.repeat(np.arange(F, dtype=np.int64), R["counts"].astype(np.int64))
    lower = np.bincount(rowner[rh[:, 0] < wb], minlength=F)
    c = np.bincount(mk, minlength=F)
    within = np.arange(len(mk)) - np.repeat(np.cumsum(c) - c, c)
    pos = roffs[mk] + lower[mk] + within
    ok &= bool(len(pos) == 0 or (pos.max() < len(rh) and np.array_equal(rh[pos], mine_h)))
    print(f"rank {rank}: subset workers {mine} holders {len(mine_h)} ok={ok}", flush=True)
    t = torch.tensor([1 if ok else 0], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MIN)
    if rank == 0:
        print("c5_check", "OK" if int(t) == 1 else "FAILED", "world", world, "F", F, "E", E, "N", N)
    dp.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
