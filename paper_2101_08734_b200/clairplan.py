"""Python host mirror of the clairsim hot-path API over the clairplan C ABI.

The reference (clairsim, C++) exposes the clairvoyant plan build as free functions in
``namespace clairsim`` (proj/include/clairsim/access.hpp:53-77, policies.hpp:49-90).  This
module mirrors those names, argument meanings and error behaviour (``ValueError`` with the
reference's ``std::invalid_argument`` text) on top of ``libclairplan.so``; the C++ shim
``csrc/compat/clairsim_compat.cpp`` does the same for C++ callers.

Every compute call runs on the GPU; when the CUDA library or device is missing the calls
raise (there is no CPU fallback).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libclairplan.so")

u32p = C.POINTER(C.c_uint32)
u64p = C.POINTER(C.c_uint64)
f64p = C.POINTER(C.c_double)

OK, ENOMEM, ENODEV, EINVAL, ERANGE, EOVERFLOW, ECUDA, ENCCL = 0, 12, 19, 22, 34, 75, 1001, 1002


class ClairplanError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


class _Config(C.Structure):
    _fields_ = [
        ("seed", C.c_uint64),
        ("samples", C.c_uint32),
        ("num_workers", C.c_uint32),
        ("global_batch", C.c_uint32),
        ("epochs", C.c_uint32),
        ("drop_last", C.c_int32),
        ("num_classes", C.c_uint32),
        ("capacities_mb", f64p),
        ("sizes_mb", f64p),
        ("sizes_on_device", C.c_int32),
        ("device", C.c_int32),
        ("worker_begin", C.c_uint32),
        ("worker_end", C.c_uint32),
    ]


class _Stats(C.Structure):
    _fields_ = [
        ("accesses", C.c_uint64),
        ("pairs", C.c_uint64),
        ("holders", C.c_uint64),
        ("rejections", C.c_uint64),
        ("device_ms", C.c_double),
        ("path", C.c_uint32),
        ("reserved", C.c_uint32),
    ]


_lib = None


def lib():
    """Load libclairplan.so (raises if it was not built: no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise FileNotFoundError(f"{LIB_PATH} missing: run __graft_entry__.build()")
    L = C.CDLL(LIB_PATH)
    L.clairplan_last_error.restype = C.c_char_p
    L.clairplan_version.restype = C.c_int
    L.clairplan_validate.argtypes = [C.POINTER(_Config)]
    L.clairplan_create.argtypes = [C.POINTER(_Config), C.POINTER(C.c_void_p)]
    L.clairplan_destroy.argtypes = [C.c_void_p]
    L.clairplan_build.argtypes = [C.c_void_p]
    L.clairplan_stats_get.argtypes = [C.c_void_p, C.POINTER(_Stats)]
    L.clairplan_launch_count.argtypes = [C.c_void_p]
    L.clairplan_launch_count.restype = C.c_uint64
    L.clairplan_device_streams.argtypes = [C.c_void_p, C.POINTER(u32p), u64p]
    L.clairplan_stream_offset.argtypes = [C.c_void_p, C.c_uint32]
    L.clairplan_stream_offset.restype = C.c_uint64
    L.clairplan_class_list_bounds.argtypes = [C.c_void_p, u64p, u64p]
    L.clairplan_device_class_lists.argtypes = [C.c_void_p, C.POINTER(u32p)]
    L.clairplan_device_holders.argtypes = [C.c_void_p, C.POINTER(u64p), C.POINTER(u32p), u64p]
    L.clairplan_export_stream.argtypes = [C.c_void_p, C.c_uint32, u32p, C.c_uint64, u64p]
    L.clairplan_export_streams.argtypes = [C.c_void_p, u32p, C.c_uint64]
    L.clairplan_export_class_lists.argtypes = [C.c_void_p, u32p, C.c_uint64]
    L.clairplan_export_holders.argtypes = [C.c_void_p, u64p, u32p, C.c_uint64]
    L.clairplan_export_counts.argtypes = [C.c_void_p, C.c_uint32, u32p]
    L.clairplan_epoch_permutation.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32, u32p, C.c_int]
    L.clairplan_access_frequencies.argtypes = [u32p, u64p, C.c_uint32, C.c_uint32, C.c_uint32,
                                               C.c_uint32, u32p, C.c_int]
    L.clairplan_worker_access_counts.argtypes = [C.POINTER(_Config), C.c_uint32, u32p]
    L.clairplan_all_access_counts.argtypes = [C.POINTER(_Config), u32p]
    L.clairplan_assign_from_streams.argtypes = [C.c_uint32, C.c_uint32, u32p, u64p, u32p,
                                                C.c_uint32, f64p, f64p, C.c_int,
                                                C.POINTER(C.c_void_p)]
    L.clairplan_reassign.argtypes = [C.c_void_p, f64p]
    L.clairplan_build_index.argtypes = [C.c_uint32, C.c_uint32, C.c_uint64, u32p, u64p, u64p,
                                        u32p, C.c_int]
    L.clairplan_generate_sizes.argtypes = [C.c_uint64, C.c_double, C.c_double, C.c_int,
                                           C.c_double, C.c_uint64, C.c_int, f64p]
    L.clairplan_choose_sources.argtypes = [C.c_void_p, C.c_uint64, u32p, u32p, u64p, f64p, f64p,
                                           C.c_double, C.c_int, C.c_int, C.c_int, C.c_int,
                                           C.c_void_p]
    L.clairplan_earliest_holders.argtypes = [C.c_void_p, f64p, u32p]
    L.clairplan_wire_size.argtypes = [C.c_void_p, u64p]
    L.clairplan_wire_write.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64]
    L.clairplan_count_histogram.argtypes = [C.c_void_p, C.c_uint32, C.c_uint32, u64p]
    L.clairplan_monte_carlo_histogram.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32,
                                                  u64p, C.c_int]
    L.clairplan_count_extremes.argtypes = [C.POINTER(_Config), u32p, u32p]
    _lib = L
    return L


# clairplan_source (include/clairplan.h): kind = FetchSource::Kind (0 Pfs, 1 Remote, 2 Local)
SOURCE_DTYPE = np.dtype([("kind", np.uint8), ("storage_class", np.uint8), ("reserved", np.uint16),
                         ("worker", np.uint32)])
SRC_PFS, SRC_REMOTE, SRC_LOCAL = 0, 1, 2


def _check(rc: int) -> None:
    if rc == OK:
        return
    msg = lib().clairplan_last_error().decode()
    if rc == EINVAL:
        raise ValueError(msg)  # std::invalid_argument in the reference
    raise ClairplanError(rc, msg)


def _p(a, t):
    return a.ctypes.data_as(t)


# ----------------------------------------------------------------- reference value types
@dataclass
class PartitionSpec:
    """access.hpp:19-28"""
    num_workers: int = 1
    global_batch: int = 1
    epochs: int = 1
    drop_last: bool = True


@dataclass
class AccessStream:
    """access.hpp:32-43 (entries + epoch/batch offsets)."""
    worker_id: int = 0
    entries: np.ndarray = field(default_factory=lambda: np.empty(0, np.uint32))
    epoch_offsets: np.ndarray = field(default_factory=lambda: np.zeros(1, np.uint64))
    batch_offsets: np.ndarray = field(default_factory=lambda: np.zeros(1, np.uint64))

    def epoch_count(self) -> int:
        return len(self.epoch_offsets) - 1

    def epoch_entries(self, e: int) -> np.ndarray:
        return self.entries[int(self.epoch_offsets[e]):int(self.epoch_offsets[e + 1])]


@dataclass
class FrequencyTable:
    """access.hpp:46-49"""
    worker_id: int = 0
    counts: np.ndarray = field(default_factory=lambda: np.empty(0, np.uint32))


@dataclass
class CacheAssignment:
    """policies.hpp:49-70: class_lists[w][j-1], holder CSR (u64 offsets here)."""
    class_lists: list = field(default_factory=list)
    holder_offsets: np.ndarray = field(default_factory=lambda: np.empty(0, np.uint64))
    holders: np.ndarray = field(default_factory=lambda: np.empty((0, 3), np.uint32))

    def empty(self) -> bool:
        return len(self.holders) == 0

    def holders_of(self, sample: int) -> np.ndarray:
        if len(self.holder_offsets) == 0:
            return self.holders[:0]
        return self.holders[int(self.holder_offsets[sample]):int(self.holder_offsets[sample + 1])]

    def build_index(self, samples: int, device: int = 0) -> None:
        """policies.cpp:124-142 — rebuilds the CSR on the GPU from (edited) class lists."""
        N = len(self.class_lists)
        J = len(self.class_lists[0]) if N else 0
        lens = [len(l) for lists in self.class_lists for l in lists]
        off = np.zeros(N * J + 1, np.uint64)
        off[1:] = np.cumsum(lens) if lens else []
        flat = np.ascontiguousarray(np.concatenate([np.asarray(l, np.uint32) for lists in
                                                    self.class_lists for l in lists])
                                    if lens else np.empty(0, np.uint32), np.uint32)
        offs = np.empty(samples + 1, np.uint64)
        hold = np.empty(max(len(flat), 1) * 3, np.uint32)
        _check(lib().clairplan_build_index(N, J, samples, _p(flat, u32p) if len(flat) else None,
                                           _p(off, u64p), _p(offs, u64p), _p(hold, u32p), device))
        self.holder_offsets = offs
        self.holders = hold[:len(flat) * 3].reshape(len(flat), 3)


# ----------------------------------------------------------------- the device plan
class Plan:
    """One device-resident plan (clairplan_t).  ``build()`` runs the whole hot path."""

    def __init__(self, seed: int, samples: int, part: PartitionSpec, capacities_mb,
                 sizes_mb, device: int = 0, worker_range=None, sizes_device_ptr: int = 0):
        self._h = C.c_void_p()
        caps = np.ascontiguousarray(capacities_mb, np.float64)
        self._caps = caps
        cfg = _Config()
        cfg.seed = seed
        cfg.samples = samples
        cfg.num_workers = part.num_workers
        cfg.global_batch = part.global_batch
        cfg.epochs = part.epochs
        cfg.drop_last = int(part.drop_last)
        cfg.num_classes = len(caps)
        cfg.capacities_mb = _p(caps, f64p) if len(caps) else None
        if sizes_device_ptr:
            cfg.sizes_mb = C.cast(C.c_void_p(sizes_device_ptr), f64p)
            cfg.sizes_on_device = 1
        else:
            sz = np.ascontiguousarray(sizes_mb, np.float64)
            self._sizes = sz
            cfg.sizes_mb = _p(sz, f64p)
        cfg.device = device
        if worker_range is not None:
            cfg.worker_begin, cfg.worker_end = worker_range
        self.cfg = cfg
        self.samples, self.part, self.J = samples, part, len(caps)
        self.wbegin = cfg.worker_begin if worker_range else 0
        self.wend = cfg.worker_end if worker_range else part.num_workers
        _check(lib().clairplan_create(C.byref(cfg), C.byref(self._h)))

    def close(self):
        if self._h:
            lib().clairplan_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def build(self) -> "Plan":
        _check(lib().clairplan_build(self._h))
        return self

    def reassign(self, capacities_mb) -> "Plan":
        """New cache-class capacities on the built plan (sweep re-planning): reruns first fit,
        prefetch orders and holders only."""
        caps = np.ascontiguousarray(capacities_mb, np.float64)
        if len(caps) != self.J:
            raise ValueError("the number of cache classes is fixed at creation")
        self._caps = caps
        _check(lib().clairplan_reassign(self._h, _p(caps, f64p) if len(caps) else None))
        return self

    def stats(self) -> dict:
        s = _Stats()
        _check(lib().clairplan_stats_get(self._h, C.byref(s)))
        return {"accesses": s.accesses, "pairs": s.pairs, "holders": s.holders,
                "rejections": s.rejections, "device_ms": s.device_ms,
                "path": {0: "v1", 1: "tier", 2: "allfit"}.get(s.path, str(s.path))}

    def launch_count(self) -> int:
        return int(lib().clairplan_launch_count(self._h))

    # ---- device views (raw pointers, for torch / cuda-python consumers)
    def device_streams(self):
        ptr, n = u32p(), C.c_uint64()
        _check(lib().clairplan_device_streams(self._h, C.byref(ptr), C.byref(n)))
        return C.cast(ptr, C.c_void_p).value, n.value

    def device_holders(self):
        po, ph, n = u64p(), u32p(), C.c_uint64()
        _check(lib().clairplan_device_holders(self._h, C.byref(po), C.byref(ph), C.byref(n)))
        return C.cast(po, C.c_void_p).value, C.cast(ph, C.c_void_p).value, n.value

    # ---- host export
    def stream(self, w: int) -> np.ndarray:
        n = int(lib().clairplan_stream_offset(self._h, w + 1) -
                lib().clairplan_stream_offset(self._h, w))
        out = np.empty(max(n, 1), np.uint32)
        ln = C.c_uint64()
        _check(lib().clairplan_export_stream(self._h, w, _p(out, u32p), n, C.byref(ln)))
        return out[:n]

    def streams_flat(self) -> np.ndarray:
        _, n = self.device_streams()
        out = np.empty(max(n, 1), np.uint32)
        _check(lib().clairplan_export_streams(self._h, _p(out, u32p), n))
        return out[:n]

    def class_lists(self):
        nloc, J = self.wend - self.wbegin, self.J
        off = np.zeros(max(nloc * J, 1), np.uint64)
        ln = np.zeros(max(nloc * J, 1), np.uint64)
        _check(lib().clairplan_class_list_bounds(self._h, _p(off, u64p), _p(ln, u64p)))
        total = int(ln[:nloc * J].sum())
        flat = np.empty(max(total, 1), np.uint32)
        _check(lib().clairplan_export_class_lists(self._h, _p(flat, u32p), total))
        out, o = [], 0
        for w in range(nloc):
            row = []
            for j in range(J):
                n = int(ln[w * J + j])
                row.append(flat[o:o + n].copy())
                o += n
            out.append(row)
        return out

    def holders(self):
        _, _, H = self.device_holders()
        offs = np.empty(self.samples + 1, np.uint64)
        hold = np.empty(max(H, 1) * 3, np.uint32)
        _check(lib().clairplan_export_holders(self._h, _p(offs, u64p), _p(hold, u32p), H))
        return offs, hold[:H * 3].reshape(H, 3)

    def counts(self, w: int) -> np.ndarray:
        out = np.empty(self.samples, np.uint32)
        _check(lib().clairplan_export_counts(self._h, w, _p(out, u32p)))
        return out

    def assignment(self) -> CacheAssignment:
        offs, hold = self.holders()
        return CacheAssignment(self.class_lists(), offs, hold)

    def choose_sources(self, samples, workers, progress, local_time, remote_time, pfs_time,
                       allow_local=True, allow_remote=True, heuristic=False) -> np.ndarray:
        """choose_source / nopfs_choose_source (policies.cpp:184-233) for every (sample, worker)
        query at once over this plan's holder CSR.  progress[w, j] = completed prefetches of
        worker w in class j + 1 (PrefetchProgress, all N workers); local_time / remote_time[j]
        and pfs_time: the unit fetch times of the caller's SystemConfig (perfmodel.cpp:109-121).
        Returns a SOURCE_DTYPE array (kind, storage_class, worker)."""
        samples = np.ascontiguousarray(samples, np.uint32)
        workers = np.ascontiguousarray(workers, np.uint32)
        progress = np.ascontiguousarray(progress, np.uint64)
        lt = np.ascontiguousarray(local_time, np.float64)
        rt = np.ascontiguousarray(remote_time, np.float64)
        if samples.shape != workers.shape:
            raise ValueError("samples and workers must have the same length")
        out = np.zeros(len(samples), SOURCE_DTYPE)
        _check(lib().clairplan_choose_sources(self._h, len(samples), _p(samples, u32p),
                                              _p(workers, u32p), _p(progress, u64p), _p(lt, f64p),
                                              _p(rt, f64p), float(pfs_time), int(allow_local),
                                              int(allow_remote), int(heuristic), 0,
                                              out.ctypes.data_as(C.c_void_p)))
        return out

    def wire(self) -> np.ndarray:
        """The plan as a versioned binary image (include/clairplan.h, wire.py parses it)."""
        n = C.c_uint64()
        _check(lib().clairplan_wire_size(self._h, C.byref(n)))
        out = np.empty(n.value, np.uint8)
        _check(lib().clairplan_wire_write(self._h, out.ctypes.data_as(C.c_void_p), n.value))
        return out

    def count_histogram(self, worker: int, max_count: int) -> np.ndarray:
        """FrequencyHistogram of `worker`'s access counts, computed on the device."""
        out = np.zeros(max_count + 1, np.uint64)
        _check(lib().clairplan_count_histogram(self._h, worker, max_count, _p(out, u64p)))
        return out

    def earliest_holders(self, remote_time) -> np.ndarray:
        """Per sample the holder {worker, class, position} with the smallest (remote unit fetch
        time, position, worker): the north star's "earliest remote holder" table (a derived view;
        0xFFFFFFFF rows for samples nobody caches)."""
        rt = np.ascontiguousarray(remote_time, np.float64)
        out = np.empty(self.samples * 3, np.uint32)
        _check(lib().clairplan_earliest_holders(self._h, _p(rt, f64p), _p(out, u32p)))
        return out.reshape(self.samples, 3)


class StreamsAssignment(Plan):
    """Handle created by clairplan_assign_from_streams (nopfs_assign_caches semantics)."""

    def __init__(self, handle, samples, N, J):
        self._h = handle
        self.samples, self.J = samples, J
        self.wbegin, self.wend = 0, N


# ----------------------------------------------------------------- clairsim mirror
def batch_slice(batch_size: int, workers: int, worker: int):
    """access.cpp:33-39 (host arithmetic)."""
    base, extra = batch_size // workers, batch_size % workers
    begin = worker * base + min(worker, extra)
    return begin, begin + base + (1 if worker < extra else 0)


def _cfg_only(seed, samples, part: PartitionSpec, device=0) -> _Config:
    cfg = _Config()
    cfg.seed, cfg.samples = seed, samples
    cfg.num_workers, cfg.global_batch = part.num_workers, part.global_batch
    cfg.epochs, cfg.drop_last = part.epochs, int(part.drop_last)
    cfg.device = device
    dummy = np.zeros(1, np.float64)
    cfg.sizes_mb = _p(dummy, f64p)
    cfg._keep = dummy
    return cfg


def validate(part: PartitionSpec, samples: int) -> None:
    """PartitionSpec::validate (access.cpp:41-50)."""
    _check(lib().clairplan_validate(C.byref(_cfg_only(0, samples, part))))


def epoch_permutation(seed: int, epoch: int, samples: int, device: int = 0) -> np.ndarray:
    """access.hpp:58 — bit-exact with the reference, computed on the GPU."""
    out = np.empty(max(samples, 1), np.uint32)
    _check(lib().clairplan_epoch_permutation(seed, epoch, samples, _p(out, u32p), device))
    return out[:samples]


def _offsets(part: PartitionSpec, samples: int, w: int):
    full = samples // part.global_batch
    tail = 0 if part.drop_last else samples % part.global_batch
    lens = [batch_slice(part.global_batch, part.num_workers, w)] * full
    if tail:
        lens.append(batch_slice(tail, part.num_workers, w))
    per = np.array([e - b for b, e in lens], np.uint64)
    bo = np.zeros(part.epochs * len(per) + 1, np.uint64)
    bo[1:] = np.cumsum(np.tile(per, part.epochs))
    eo = bo[::len(per)] if len(per) else np.zeros(part.epochs + 1, np.uint64)
    return eo.astype(np.uint64), bo


def build_access_streams(seed: int, samples: int, part: PartitionSpec, device: int = 0):
    """access.hpp:62-63 — per-worker AccessStreams (streams built on the GPU)."""
    plan = Plan(seed, samples, part, [], np.zeros(1), device=device)
    plan.build()
    out = []
    for w in range(part.num_workers):
        eo, bo = _offsets(part, samples, w)
        out.append(AccessStream(w, plan.stream(w), eo, bo))
    plan.close()
    return out


def access_frequencies(stream: AccessStream, samples: int, epoch_begin: int, epoch_end: int,
                       device: int = 0) -> FrequencyTable:
    """access.hpp:66-67"""
    ent = np.ascontiguousarray(stream.entries, np.uint32)
    eo = np.ascontiguousarray(stream.epoch_offsets, np.uint64)
    out = np.empty(samples, np.uint32)
    _check(lib().clairplan_access_frequencies(_p(ent, u32p) if len(ent) else None, _p(eo, u64p),
                                              stream.epoch_count(), samples, epoch_begin,
                                              epoch_end, _p(out, u32p), device))
    return FrequencyTable(stream.worker_id, out)


def worker_access_counts(seed: int, samples: int, part: PartitionSpec, worker: int,
                         device: int = 0) -> np.ndarray:
    """access.hpp:71-72"""
    out = np.empty(samples, np.uint32)
    _check(lib().clairplan_worker_access_counts(C.byref(_cfg_only(seed, samples, part, device)),
                                                worker, _p(out, u32p)))
    return out


def all_access_counts(seed: int, samples: int, part: PartitionSpec, device: int = 0) -> np.ndarray:
    """access.hpp:76-77 -> [N][F]"""
    out = np.empty((part.num_workers, samples), np.uint32)
    _check(lib().clairplan_all_access_counts(C.byref(_cfg_only(seed, samples, part, device)),
                                             _p(out, u32p)))
    return out


def nopfs_assign_caches(freqs, capacities_mb, sizes_mb, streams, device: int = 0) -> CacheAssignment:
    """policies.hpp:88-90 on explicit streams and frequency tables (the drop-in form)."""
    N = len(freqs)
    F = len(sizes_mb)
    counts = np.ascontiguousarray(np.stack([np.asarray(f.counts, np.uint32) for f in freqs]))
    ent = np.ascontiguousarray(np.concatenate([s.entries for s in streams])
                               if N else np.empty(0), np.uint32)
    offs = np.zeros(N + 1, np.uint64)
    offs[1:] = np.cumsum([len(s.entries) for s in streams])
    caps = np.ascontiguousarray(capacities_mb, np.float64)
    sz = np.ascontiguousarray(sizes_mb, np.float64)
    h = C.c_void_p()
    _check(lib().clairplan_assign_from_streams(
        N, F, _p(ent, u32p) if len(ent) else None, _p(offs, u64p), _p(counts, u32p), len(caps),
        _p(caps, f64p) if len(caps) else None, _p(sz, f64p), device, C.byref(h)))
    plan = StreamsAssignment(h, F, N, len(caps))
    a = plan.assignment()
    plan.close()
    return a


def monte_carlo_histogram(seed: int, workers: int, epochs: int, samples: int,
                          device: int = 0) -> np.ndarray:
    """analysis.cpp:84-96 on the device: worker 0's count histogram (B = N, drop_last=false)."""
    out = np.zeros(epochs + 1, np.uint64)
    _check(lib().clairplan_monte_carlo_histogram(seed, workers, epochs, samples, _p(out, u64p), device))
    return out


def count_extremes(seed: int, samples: int, part: PartitionSpec, device: int = 0):
    """Per sample (largest, smallest) access count over all workers, from device counts
    (the Lemma-1 property suite's inputs, acceptance.cpp:98-158)."""
    cfg = _cfg_only(seed, samples, part, device)
    hi = np.empty(samples, np.uint32)
    lo = np.empty(samples, np.uint32)
    _check(lib().clairplan_count_extremes(C.byref(cfg), _p(hi, u32p), _p(lo, u32p)))
    return hi, lo


def generate_sizes(samples: int, mean_mb: float, sigma_mb: float, total_mb=None, seed: int = 1,
                   sigma_relative: bool = False) -> np.ndarray:
    """DatasetModel::generate (perfmodel.cpp:68-99) — host input generator."""
    out = np.empty(samples, np.float64)
    _check(lib().clairplan_generate_sizes(samples, mean_mb, sigma_mb, total_mb is not None,
                                          total_mb or 0.0, seed, int(sigma_relative),
                                          _p(out, f64p)))
    return out


# scenarios.cpp:15-46: staging 5,000 MB (class 0, not packed), RAM 120,000 MB, SSD 900,000 MB
REFERENCE_CAPACITIES_MB = (120000.0, 900000.0)
