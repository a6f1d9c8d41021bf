"""Host logic of the multi-GPU plan on CPU: world_size-2 gloo process group.

The device work of each rank is replaced by the reference's own plan restricted to the rank's
worker range (what a rank produces), so the test checks the sharding and the NCCL-side merge
(epoch ranges, padded row all-gather, holder-offset merge) against the single-process plan."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2101_08734_b200.distributed import (epoch_ranges, gather_rows,
                                               holder_offsets_from_counts,
                                               rank_offsets_from_counts, stream_splits,
                                               worker_range)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from _oracle import Port
        port_ = Port()
        seed, F, N, B, E = 3, 700, 5, 20, 7
        caps = [3.0, 6.0]
        sizes = port_.generate_sizes(F, 0.1, 0.05, None, 1)
        # 1) epoch-sharded permutation rows, padded all-gather
        ranges, pad = epoch_ranges(E, world)
        e0, n = ranges[rank]
        local = torch.tensor(np.stack([port_.epoch_permutation(seed, e, F) for e in range(e0, e0 + n)])
                             .astype(np.int32))
        rows = gather_rows(local, ranges, pad)
        full = np.stack([port_.epoch_permutation(seed, e, F) for e in range(E)]).astype(np.int32)
        ok_rows = np.array_equal(rows.numpy(), full)
        # 2) worker-sharded holder records + offset merge
        whole = port_.plan(seed, F, N, B, E, True, caps, sizes)
        wb, we = worker_range(N, rank, world)
        mine = whole.holders[(whole.holders[:, 0] >= wb) & (whole.holders[:, 0] < we)]
        owner = np.repeat(np.arange(F), np.diff(whole.holder_offsets.astype(np.int64)))
        mine_k = owner[(whole.holders[:, 0] >= wb) & (whole.holders[:, 0] < we)]
        counts = torch.tensor(np.bincount(mine_k, minlength=F).astype(np.int32))
        allc = [torch.empty_like(counts) for _ in range(world)]
        dist.all_gather(allc, counts)
        glob, starts = holder_offsets_from_counts(torch.stack(allc))
        ok_glob = np.array_equal(glob.numpy(), whole.holder_offsets.astype(np.int64))
        g2, s2 = rank_offsets_from_counts(torch.stack(allc), rank)
        ok_glob &= np.array_equal(g2.numpy(), glob.numpy()) and np.array_equal(
            s2.numpy(), starts[rank].numpy())
        # place this rank's records at their global positions: must equal the global slice
        pos = starts[rank].numpy()[mine_k] + (np.arange(len(mine_k)) -
                                             np.repeat(np.cumsum(counts.numpy()) - counts.numpy(),
                                                       counts.numpy()))
        ok_pos = np.array_equal(whole.holders[pos], mine)
        # 3) epoch-range streams of all workers -> all-to-all -> this rank's worker streams
        #    (clairplan_generate_streams / _build_from_streams layouts, relayout in numpy)
        Le = [len(st) // E for st in whole.streams]
        prefix = np.concatenate([[0], np.cumsum(Le)]).astype(np.int64)
        wr = [worker_range(N, r, world) for r in range(world)]
        send_s, recv_s = stream_splits(prefix, ranges, wr, rank)
        send = np.concatenate([whole.streams[w][e0 * Le[w]:(e0 + n) * Le[w]] for w in range(N)])
        assert len(send) == sum(send_s) == n * prefix[N]
        recv = torch.empty(sum(recv_s), dtype=torch.int32)
        dist.all_to_all_single(recv, torch.tensor(send.astype(np.int32)), recv_s, send_s)
        recv = recv.numpy()
        got, off = [], 0
        parts = {}
        for r, (er, nr) in enumerate(ranges):
            for w in range(wb, we):
                parts[(w, r)] = recv[off:off + nr * Le[w]]
                off += nr * Le[w]
        for w in range(wb, we):
            got.append(np.concatenate([parts[(w, r)] for r in range(world)]))
        ok_streams = all(np.array_equal(g, whole.streams[w].astype(np.int32))
                         for g, w in zip(got, range(wb, we)))
        q.put((rank, ok_rows and ok_streams, ok_glob, ok_pos))
    finally:
        dist.destroy_process_group()


def test_two_rank_sharding_and_merge_gloo():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    assert all(p.exitcode == 0 for p in procs)
    for rank, ok_rows, ok_glob, ok_pos in res:
        assert ok_rows and ok_glob and ok_pos, (rank, ok_rows, ok_glob, ok_pos)


def test_epoch_and_worker_ranges():
    for E in (1, 7, 90, 100):
        for world in (1, 2, 3, 8):
            ranges, pad = epoch_ranges(E, world)
            assert sum(n for _, n in ranges) == E and max(n for _, n in ranges) <= pad
            assert [b for b, _ in ranges] == list(np.cumsum([0] + [n for _, n in ranges])[:-1])
    assert [worker_range(1024, r, 8) for r in (0, 7)] == [(0, 128), (896, 1024)]
