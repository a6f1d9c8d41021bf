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


def checksum_case(rank, world, F, N, b, E, mu, sd, tot):
    import ctypes as C
    from paper_2101_08734_b200 import wire
    L = cp.lib()
    L.clairplan_wire_checksums.argtypes = [C.c_void_p, C.c_uint64, C.c_uint64, C.c_void_p,
                                           C.POINTER(C.c_uint64)]
    caps = [120_000.0, 900_000.0]
    sizes = cp.generate_sizes(F, mu, sd, tot, 1)
    part = cp.PartitionSpec(N, b * N, E, True)
    dp = DistributedPlan(42, F, part, caps, sizes).build()
    st = dp.plan.stats()
    wb, we = dp.wrange
    hloc = torch.tensor([st["holders"]], dtype=torch.int64, device="cuda")
    allh = [torch.zeros_like(hloc) for _ in range(world)]
    dist.all_gather(allh, hloc)
    list_base = int(sum(int(x) for x in allh[:rank]))
    starts = dp.rank_starts.contiguous()
    out = (C.c_uint64 * 6)()
    sb = cp.lib().clairplan_stream_offset(dp.plan._h, wb)  # = 0 for a shard; global offset below
    pre = C.c_uint64()
    cp._check(L.clairplan_epoch_prefix(dp.plan._h, wb, C.byref(pre)))
    stream_base = E * int(pre.value)
    cp._check(L.clairplan_wire_checksums(dp.plan._h, stream_base, list_base,
                                         C.c_void_p(starts.data_ptr()), out))
    mine = torch.tensor([int(x) - (1 << 64) if int(x) >= (1 << 63) else int(x) for x in out],
                        dtype=torch.int64, device="cuda")
    dist.all_reduce(mine)  # int64 sums wrap mod 2^64
    merged = [int(x) & ((1 << 64) - 1) for x in mine.cpu().tolist()]
    merged[4] = wire.section_checksum(dp.global_offsets.cpu().numpy().astype(np.uint64), 4)
    dp.close()
    full = cp.Plan(42, F, part, caps, sizes, device=torch.cuda.current_device()).build()
    ref = (C.c_uint64 * 6)()
    cp._check(L.clairplan_wire_checksums(full._h, 0, 0, None, ref))
    fst = full.stats()
    full.close()
    want = [int(x) for x in ref]
    good = all(merged[i] == want[i] for i in (1, 3, 4, 5)) and sb == 0
    print(f"rank {rank} F={F} N={N} E={E} checksums {'equal' if good else 'DIFFER'} "
          f"(path {st['path']}, local A {st['accesses']}, full D {fst['pairs']})", flush=True)
    return good


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
        c_st = np.array_equal(st_full[lo:hi], st_mine)
        # class lists of my workers
        cl_full, cl_mine = full.class_lists()[wb:we], dp.plan.class_lists()
        c_cl = all(np.array_equal(x, y) for a, c in zip(cl_full, cl_mine) for x, y in zip(a, c))
        # holder CSR: global offsets and my records at their global positions
        c_go = np.array_equal(dp.global_offsets.cpu().numpy(), offs_full.astype(np.int64))
        if not (c_st and c_cl and c_go):
            print(f"rank {rank}: streams {c_st} class lists {c_cl} global offsets {c_go} "
                  f"merged-overlapped {getattr(dp, 'merge_overlapped', None)}", flush=True)
        ok &= c_st and c_cl and c_go
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
            c_h = bool(np.array_equal(hold_full[pos], hold_mine))
            if not c_h:
                print(f"rank {rank}: holder records at global positions differ", flush=True)
            ok &= c_h
        print(f"rank {rank} F={F} N={N} E={E} dl={dl} mode={mode} ok={ok}", flush=True)
        dp.close()
        full.close()
    # benchmark-scale shapes (config 2 at 90 epochs: all-fit path; config 4: tier path, the
    # north-star shape), checked without host copies: the shards' section checksums placed at
    # their merged positions, summed over ranks, equal the single-GPU plan's (which the GPU
    # suite checks against the reference in full)
    only = os.environ.get("DIST_CHECK_BIG", "2,4")
    big = {"2": (1_281_167, 256, 32, 90, (0.1077, 0.1, 135_000.0)),
           "4": (14_197_122, 1024, 32, 90, (0.1077, 0.2, 1_500_000.0))}
    for key in [k for k in only.split(",") if k]:
        F, N, b, E, (mu, sd, tot) = big[key]
        ok &= checksum_case(rank, world, F, N, b, E, mu, sd, tot)
    t = torch.tensor([1 if ok else 0], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MIN)
    if rank == 0:
        print("dist_check", "OK" if int(t) == 1 else "FAILED", "world", world)
    dist.destroy_process_group()
    sys.exit(0 if int(t) == 1 else 1)


if __name__ == "__main__":
    main()
