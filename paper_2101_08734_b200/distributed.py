"""Multi-GPU plan build: one process per GPU, torch.distributed (NCCL) for the exchanges.

Decomposition ("Multi-GPU"):
  1. epoch sharding  — rank r draws the permutations of its epoch range and cuts them into
                       the access streams of ALL workers for those epochs
                       (clairplan_generate_streams); epochs are independent by construction
                       (access.cpp:52-57: epoch e owns stream positions [e<<34, (e+1)<<34)).
  2. all-to-all      — every rank sends each other rank the stream slices of that rank's
                       workers (one ncclAllToAll-style exchange through torch.distributed,
                       4A(G-1)/G bytes in total over NVLink).
  3. worker sharding — rank r re-lays out its workers' streams, rebuilds the inverse
                       permutations restricted to its workers and builds the (count,
                       first-access) tables, tier assignment, prefetch orders and holder
                       records of its contiguous worker range (clairplan_build_from_streams);
                       nopfs_assign_caches has no cross-worker dependency (policies.cpp:151-163).
  4. holder merge    — per-sample holder counts are all-gathered; the global CSR offset of
                       sample k is the exclusive scan of the per-sample totals and rank r's
                       records of k start after those of ranks < r (worker ranges ascend, so
                       this is build_index's worker order, policies.cpp:124-142).

The output stays sharded: rank r owns its workers' streams / class lists and its holder
records with their global CSR positions.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np


def epoch_ranges(E: int, world: int):
    """Balanced contiguous epoch ranges, one per rank; padded row count for the gather."""
    base, extra = divmod(E, world)
    ranges, b = [], 0
    for r in range(world):
        n = base + (1 if r < extra else 0)
        ranges.append((b, n))
        b += n
    return ranges, base + (1 if extra else 0)


def worker_range(N: int, rank: int, world: int):
    return rank * N // world, (rank + 1) * N // world


def holder_offsets_from_counts(counts):
    """counts: [world, F] per-rank per-sample holder counts (torch or numpy, integer).
    Returns (global_offsets[F+1], rank_starts[world, F]): the global CSR offsets and, for
    every rank, where its records of sample k start in the global holder array."""
    import torch
    c = torch.as_tensor(counts).to(torch.int64)
    tot = c.sum(dim=0)
    glob = torch.zeros(c.shape[1] + 1, dtype=torch.int64, device=c.device)
    glob[1:] = torch.cumsum(tot, dim=0)
    before = torch.cumsum(c, dim=0) - c  # exclusive over ranks
    return glob, glob[:-1].unsqueeze(0) + before


def rank_offsets_from_counts(counts, rank):
    """holder_offsets_from_counts for one rank: (global_offsets[F+1], rank_starts[F]) with a
    few kernels over the [world, F] counts (no [world, F] int64 intermediates)."""
    import torch
    tot = counts.sum(dim=0, dtype=torch.int64)
    glob = torch.zeros(counts.shape[1] + 1, dtype=torch.int64, device=counts.device)
    torch.cumsum(tot, dim=0, out=glob[1:])
    if rank == 0:
        return glob, glob[:-1]
    return glob, glob[:-1] + counts[:rank].sum(dim=0, dtype=torch.int64)


def stream_splits(prefix, ranges, wranges, rank):
    """All-to-all split sizes (u32 entries) of the epoch-range streams.
    prefix[w] = stream entries per epoch of workers < w; ranges[r] = (first epoch, count) of
    rank r; wranges[d] = worker range of rank d.  Rank `rank` sends rank d the entries of d's
    workers for its own epochs and receives from rank r r's epochs of its own workers."""
    n_me = ranges[rank][1]
    send = [n_me * (prefix[we] - prefix[wb]) for wb, we in wranges]
    wb, we = wranges[rank]
    recv = [n * (prefix[we] - prefix[wb]) for _, n in ranges]
    return send, recv


def gather_rows(local, ranges, pad, group=None):
    """All-gather per-rank permutation rows (uneven epoch ranges, padded) -> [E, F]."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    F = local.shape[1]
    buf = torch.zeros((pad, F), dtype=local.dtype, device=local.device)
    buf[: local.shape[0]] = local
    out = torch.empty((world * pad, F), dtype=local.dtype, device=local.device)
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(out, buf, group=group)
    else:  # gloo (CPU tests of the host logic)
        dist.all_gather(list(out.chunk(world)), buf, group=group)
    rows = [out[r * pad: r * pad + n] for r, (_, n) in enumerate(ranges)]
    return torch.cat(rows, dim=0).contiguous()


class DistributedPlan:
    """Sharded plan of one rank (call the same sequence on every rank).

    mode "streams" (default): epoch-range streams + all-to-all (steps 1-3 above);
    mode "perms": permutation rows all-gathered to every rank (the earlier scheme, kept for
    A/B measurements)."""

    def __init__(self, seed, samples, part, capacities_mb, sizes_mb, group=None, mode="p2p",
                 pipeline=False):
        import torch
        import torch.distributed as dist
        from . import clairplan as cp
        self.cp, self.torch, self.dist = cp, torch, dist
        self.group = group
        self.mode = mode
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.device = torch.cuda.current_device()
        self.samples, self.part = samples, part
        self.wrange = worker_range(part.num_workers, self.rank, self.world)
        self.plan = cp.Plan(seed, samples, part, capacities_mb, sizes_mb, device=self.device,
                            worker_range=self.wrange)
        self.ranges, self.pad = epoch_ranges(part.epochs, self.world)
        L = cp.lib()
        L.clairplan_generate_perms.argtypes = [C.c_void_p, C.c_uint32, C.c_uint32, C.c_void_p]
        L.clairplan_build_from_perms.argtypes = [C.c_void_p, C.c_void_p]
        L.clairplan_holder_counts.argtypes = [C.c_void_p, C.c_void_p]
        L.clairplan_generate_streams.argtypes = [C.c_void_p, C.c_uint32, C.c_uint32, C.c_void_p]
        L.clairplan_build_from_streams.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint32]
        L.clairplan_epoch_prefix.argtypes = [C.c_void_p, C.c_uint32, C.POINTER(C.c_uint64)]
        L.clairplan_merge_holder_counts.argtypes = [C.c_void_p, C.c_void_p, C.c_uint32, C.c_uint32,
                                                    C.c_void_p, C.c_void_p, C.c_void_p]
        self.L = L
        N = part.num_workers
        self.p2p = False
        if mode == "p2p":  # fused exchange through peer memory, else the all-to-all
            mode = self.mode = "streams"
            self.p2p = (dist.get_backend(group) == "nccl" and self.world <= 16 and
                        bool(L.clairplan_p2p_supported(self.plan._h)))
        if mode == "streams":
            pre = []
            for w in range(N + 1):
                v = C.c_uint64()
                cp._check(L.clairplan_epoch_prefix(self.plan._h, w, C.byref(v)))
                pre.append(int(v.value))
            wr = [worker_range(N, r, self.world) for r in range(self.world)]
            self.send_splits, self.recv_splits = stream_splits(pre, self.ranges, wr, self.rank)
            if self.p2p:
                self.p2p = self._setup_p2p(pre, wr)
            self.pipeline = pipeline and dist.get_backend(group) == "nccl" and not self.p2p
            self.send = None if (self.pipeline or self.p2p) else torch.empty(
                max(sum(self.send_splits), 1), dtype=torch.int32, device="cuda")
            self.recv = None if self.p2p else torch.empty(max(sum(self.recv_splits), 1),
                                                          dtype=torch.int32, device="cuda")
            self.bounds = np.array([b for b, _ in self.ranges] + [part.epochs], np.uint32)
            # pipelined variant (NCCL): every rank's epochs in two halves, the first half's
            # all-to-all overlapping the second half's shuffle (measured at 4 ranks: generate +
            # exchange 1.31 vs 1.21 ms unpipelined — the exchange competes for SMs — so off by
            # default)
            if self.pipeline:
                wb, we = self.wrange
                lloc = pre[we] - pre[wb]
                self.halves = [[(b, (n + 1) // 2), (b + (n + 1) // 2, n - (n + 1) // 2)]
                               for b, n in self.ranges]
                self.bounds2 = np.array([c[0] for h in self.halves for c in h] + [part.epochs],
                                        np.uint32)
                mine = self.halves[self.rank]
                self.send_h = [torch.empty(max(n * pre[N], 1), dtype=torch.int32, device="cuda")
                               for _, n in mine]
                self.in_lists, self.out_lists = [], []
                for h, (_, n) in enumerate(mine):
                    ins, o = [], 0
                    for (db, de) in wr:
                        ln = n * (pre[de] - pre[db])
                        ins.append(self.send_h[h][o:o + ln])
                        o += ln
                    outs = []
                    for r in range(self.world):
                        cb, cn = self.halves[r][h]
                        outs.append(self.recv[cb * lloc:(cb + cn) * lloc])
                    self.in_lists.append(ins)
                    self.out_lists.append(outs)
        else:
            self.pipeline = False
            self.local_rows = torch.empty((max(self.pad, 1), samples), dtype=torch.int32,
                                          device="cuda")
        self.counts = torch.empty(samples, dtype=torch.int32, device="cuda")
        self.allc = torch.empty((self.world, samples), dtype=torch.int32, device="cuda")
        # holder-offset merge overlapped with the build's tail (streams mode, NCCL): the
        # library calls _on_counts once the pair counts exist; its all-gather runs while the
        # all-fit kernels finish.  Valid when every rank's build took the all-fit path.
        self._spec = None
        self._hook = None
        L.clairplan_set_counts_hook.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                                C.c_void_p]
        L.clairplan_counts_hook_valid.argtypes = [C.c_void_p]
        if mode == "streams" and dist.get_backend(group) == "nccl" and \
                os.environ.get("CLAIRPLAN_MERGE_OVERLAP", "1") != "0":
            self._hook = C.CFUNCTYPE(None, C.c_void_p)(self._on_counts)
            cp._check(L.clairplan_set_counts_hook(
                self.plan._h, C.c_void_p(self.counts.data_ptr()),
                C.c_void_p(torch.cuda.current_stream().cuda_stream),
                C.cast(self._hook, C.c_void_p), None))
        self.timings = {}
        self.global_offsets = None
        self.rank_starts = None

    def _setup_p2p(self, pre, wr):
        """Two receive buffers per rank (alternating builds), their CUDA IPC handles exchanged
        once; every rank's shuffle then writes each stream entry into its owner's buffer.
        Collective and all-or-nothing: returns False on every rank (all-to-all fallback) if
        any rank could not allocate, export or open a buffer."""
        torch, L, cp = self.torch, self.L, self.cp
        L.clairplan_recv_buffer.argtypes = [C.c_void_p, C.c_uint32, C.POINTER(C.c_void_p), C.c_void_p]
        L.clairplan_open_peer_buffer.argtypes = [C.c_void_p, C.c_void_p, C.POINTER(C.c_void_p)]
        L.clairplan_generate_streams_p2p.argtypes = [C.c_void_p, C.c_uint32, C.c_uint32, C.c_void_p,
                                                     C.c_void_p, C.c_void_p, C.c_uint32]
        own, handles = [], []
        try:
            for i in range(2):
                ptr, hb = C.c_void_p(), (C.c_char * 64)()
                cp._check(L.clairplan_recv_buffer(self.plan._h, i, C.byref(ptr), hb))
                own.append(ptr.value)
                handles.append(bytes(hb))
        except Exception:
            handles = None
        allh = [None] * self.world
        self.dist.all_gather_object(allh, handles, group=self.group)
        ok = all(h is not None for h in allh)
        self.dst_ptrs = [np.zeros(self.world, np.uint64) for _ in range(2)]
        if ok:
            try:
                for r in range(self.world):
                    for i in range(2):
                        if r == self.rank:
                            self.dst_ptrs[i][r] = own[i]
                        else:
                            hb = (C.c_char * 64).from_buffer_copy(allh[r][i])
                            ptr = C.c_void_p()
                            cp._check(L.clairplan_open_peer_buffer(self.plan._h, hb, C.byref(ptr)))
                            self.dst_ptrs[i][r] = ptr.value
            except Exception:
                ok = False
        flag = torch.tensor([1 if ok else 0], dtype=torch.int32, device="cuda")
        self.dist.all_reduce(flag, op=self.dist.ReduceOp.MIN, group=self.group)
        if int(flag.item()) == 0:
            return False
        self.own_recv = own
        e0, ne = self.ranges[self.rank]
        # rank d's buffer holds, from this rank, [d's worker w][my epoch e][Le(w)] at e0 * lloc(d)
        self.deltas = np.array([e0 * (pre[we] - pre[wb]) - ne * pre[wb] for wb, we in wr], np.int64)
        self.wbounds = np.array([wb for wb, _ in wr] + [self.part.num_workers], np.uint32)
        self.iter = 0
        self.flag = torch.zeros(1, dtype=torch.int32, device="cuda")
        return True

    def _merge(self):
        """Global CSR offsets + this rank's starts from the gathered counts: one library call
        (merge kernel + scan) on torch's current stream, after the all-gather."""
        torch = self.torch
        glob = torch.empty(self.samples + 1, dtype=torch.int64, device="cuda")
        starts = torch.empty(self.samples, dtype=torch.int64, device="cuda")
        self.cp._check(self.L.clairplan_merge_holder_counts(
            self.plan._h, C.c_void_p(self.allc.data_ptr()), self.world, self.rank,
            C.c_void_p(glob.data_ptr()), C.c_void_p(starts.data_ptr()),
            C.c_void_p(torch.cuda.current_stream().cuda_stream)))
        return glob, starts

    def _on_counts(self, _user):
        # runs inside the library's build call (same thread); the stream already waits for the
        # counts copy
        self.dist.all_gather_into_tensor(self.allc, self.counts, group=self.group)
        self._spec = self._merge()

    def build(self):
        import time
        torch, cp = self.torch, self.cp
        e0, n = self.ranges[self.rank]
        self._spec = None
        t0 = time.perf_counter()
        if self.mode == "streams" and self.pipeline:
            works = []
            for h, (hb, hn) in enumerate(self.halves[self.rank]):
                cp._check(self.L.clairplan_generate_streams(self.plan._h, hb, hn,
                                                            C.c_void_p(self.send_h[h].data_ptr())))
                works.append(self.dist.all_to_all(self.out_lists[h], self.in_lists[h],
                                                  group=self.group, async_op=True))
            t1 = time.perf_counter()
            for wk in works:
                wk.wait()
            torch.cuda.current_stream().synchronize()
            t2 = time.perf_counter()
            cp._check(self.L.clairplan_build_from_streams(
                self.plan._h, C.c_void_p(self.recv.data_ptr()),
                self.bounds2.ctypes.data_as(C.c_void_p), 2 * self.world))
            t3 = time.perf_counter()
            self.timings = {"generate_ms": round((t1 - t0) * 1e3, 3),
                            "all_to_all_ms": round((t2 - t1) * 1e3, 3),
                            "build_ms": round((t3 - t2) * 1e3, 3)}
        elif self.mode == "streams" and self.p2p:
            i = self.iter & 1
            self.iter += 1
            cp._check(self.L.clairplan_generate_streams_p2p(
                self.plan._h, e0, n, self.dst_ptrs[i].ctypes.data_as(C.c_void_p),
                self.deltas.ctypes.data_as(C.c_void_p), self.wbounds.ctypes.data_as(C.c_void_p),
                self.world))
            t1 = time.perf_counter()
            # every rank's shuffle has finished writing into the peers' buffers (the library
            # synchronised its stream): one small all-reduce orders them before the builds
            self.dist.all_reduce(self.flag, group=self.group)
            torch.cuda.current_stream().synchronize()
            t2 = time.perf_counter()
            cp._check(self.L.clairplan_build_from_streams(
                self.plan._h, C.c_void_p(self.own_recv[i]),
                self.bounds.ctypes.data_as(C.c_void_p), self.world))
            t3 = time.perf_counter()
            self.timings = {"generate_ms": round((t1 - t0) * 1e3, 3),
                            "all_to_all_ms": round((t2 - t1) * 1e3, 3),
                            "build_ms": round((t3 - t2) * 1e3, 3)}
        elif self.mode == "streams":
            cp._check(self.L.clairplan_generate_streams(self.plan._h, e0, n,
                                                        C.c_void_p(self.send.data_ptr())))
            t1 = time.perf_counter()
            # the library synchronises its stream before returning; NCCL runs on torch's
            self.dist.all_to_all_single(self.recv[:sum(self.recv_splits)],
                                        self.send[:sum(self.send_splits)],
                                        self.recv_splits, self.send_splits, group=self.group)
            torch.cuda.current_stream().synchronize()
            t2 = time.perf_counter()
            cp._check(self.L.clairplan_build_from_streams(
                self.plan._h, C.c_void_p(self.recv.data_ptr()),
                self.bounds.ctypes.data_as(C.c_void_p), self.world))
            t3 = time.perf_counter()
            self.timings = {"generate_ms": round((t1 - t0) * 1e3, 3),
                            "all_to_all_ms": round((t2 - t1) * 1e3, 3),
                            "build_ms": round((t3 - t2) * 1e3, 3)}
        else:
            cp._check(self.L.clairplan_generate_perms(self.plan._h, e0, n,
                                                      C.c_void_p(self.local_rows.data_ptr())))
            perms = gather_rows(self.local_rows[:n], self.ranges, self.pad, self.group)
            # the gather and the concatenation run on torch's stream; the library reads the
            # rows on its own stream, so order them (every library call synchronises its own
            # stream before returning, so the reverse direction needs nothing)
            torch.cuda.current_stream().synchronize()
            cp._check(self.L.clairplan_build_from_perms(self.plan._h,
                                                        C.c_void_p(perms.data_ptr())))
            del perms
        t4 = time.perf_counter()
        merged = False
        if self._hook is not None:
            # the overlapped merge holds only if every rank's hooked counts are its holder counts
            ok = torch.tensor([1 if (self._spec is not None and
                                     self.L.clairplan_counts_hook_valid(self.plan._h)) else 0],
                              dtype=torch.int32, device="cuda")
            self.dist.all_reduce(ok, op=self.dist.ReduceOp.MIN, group=self.group)
            if int(ok.item()) == 1:
                self.global_offsets, self.rank_starts = self._spec
                merged = True
        if not merged:
            cp._check(self.L.clairplan_holder_counts(self.plan._h,
                                                     C.c_void_p(self.counts.data_ptr())))
            self.dist.all_gather_into_tensor(self.allc, self.counts, group=self.group)
            self.global_offsets, self.rank_starts = self._merge()
        self.merge_overlapped = merged
        if self.mode == "streams":
            torch.cuda.current_stream().synchronize()
            self.timings["merge_ms"] = round((time.perf_counter() - t4) * 1e3, 3)
        return self

    def stats(self):
        return self.plan.stats()

    def close(self):
        self.plan.close()
