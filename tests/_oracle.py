"""ctypes bindings to the CPU oracle (TEST INFRASTRUCTURE ONLY).

* ``Port`` loads ``oracle/libclairplan_oracle.so`` — the plain-C restatement.
* ``Ref``  loads ``oracle/_ref/libclairsim_ref.so`` — the unmodified reference sources
  plus ``oracle/ref_harness.cpp``.

Both expose the same high-level results (numpy arrays) so tests can compare the CUDA
path against either.  Nothing under ``paper_2101_08734_b200/`` imports this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE = os.path.join(ROOT, "oracle")
PORT_SO = os.path.join(ORACLE, "libclairplan_oracle.so")
REF_SO = os.path.join(ORACLE, "_ref", "libclairsim_ref.so")

u32p = C.POINTER(C.c_uint32)
u64p = C.POINTER(C.c_uint64)
f64p = C.POINTER(C.c_double)

PERM_TAG = 0x7065726D
SIZE_TAG = 0x73697A65


def _ptr(a, t):
    return a.ctypes.data_as(t)


def ensure_built(ref: bool = True) -> None:
    targets = ["port"] + (["ref"] if ref and os.path.isdir("/root/reference/proj") else [])
    if not os.path.exists(PORT_SO) or (ref and not os.path.exists(REF_SO)):
        subprocess.run(["make", "-s", "-C", ORACLE] + targets, check=True)


class Plan:
    """Host result of one plan build: streams, class lists, holder CSR (numpy)."""

    def __init__(self, N, J, streams, class_lists, holder_offsets, holders):
        self.N, self.J = N, J
        self.streams = streams              # list[N] of u32 arrays
        self.class_lists = class_lists      # [N][J] of u32 arrays
        self.holder_offsets = holder_offsets  # u64[F+1]
        self.holders = holders              # u32[H, 3] (worker, class, position)


class Port:
    def __init__(self):
        ensure_built(ref=False)
        L = C.CDLL(PORT_SO)
        L.orc_mix64.restype = C.c_uint64
        L.orc_mix64.argtypes = [C.c_uint64]
        L.orc_derive_key.restype = C.c_uint64
        L.orc_derive_key.argtypes = [C.c_uint64, C.c_uint64]
        L.orc_bounded.restype = C.c_uint64
        L.orc_bounded.argtypes = [C.c_uint64, u64p, C.c_uint64]
        L.orc_epoch_permutation.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32, u32p]
        L.orc_epoch_permutation_norej.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32, u32p]
        L.orc_generate_sizes.argtypes = [C.c_uint64, C.c_double, C.c_double, C.c_int,
                                         C.c_double, C.c_uint64, C.c_int, f64p]
        L.orc_plan_build.restype = C.c_void_p
        L.orc_plan_build.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32,
                                     C.c_int, C.c_uint32, f64p, f64p]
        L.orc_assign_from_streams.restype = C.c_void_p
        L.orc_assign_from_streams.argtypes = [C.c_uint32, C.c_uint32, u32p, u64p, u32p,
                                              C.c_uint32, f64p, f64p]
        L.orc_plan_stream.restype = C.c_uint64
        L.orc_plan_stream.argtypes = [C.c_void_p, C.c_uint32, C.POINTER(u32p)]
        L.orc_plan_class_list.restype = C.c_uint64
        L.orc_plan_class_list.argtypes = [C.c_void_p, C.c_uint32, C.c_uint32, C.POINTER(u32p)]
        L.orc_plan_holders.restype = C.c_uint64
        L.orc_plan_holders.argtypes = [C.c_void_p, C.POINTER(u64p), C.POINTER(u32p)]
        L.orc_plan_free.argtypes = [C.c_void_p]
        L.orc_last_error.restype = C.c_char_p
        self.L = L

    def epoch_permutation(self, seed, epoch, F):
        out = np.empty(F, np.uint32)
        rc = self.L.orc_epoch_permutation(seed, epoch, F, _ptr(out, u32p))
        if rc:
            raise ValueError(self.L.orc_last_error().decode())
        return out

    def epoch_permutation_norej(self, seed, epoch, F):
        out = np.empty(F, np.uint32)
        self.L.orc_epoch_permutation_norej(seed, epoch, F, _ptr(out, u32p))
        return out

    def generate_sizes(self, F, mean, sigma, total=None, seed=1, sigma_relative=False):
        out = np.empty(F, np.float64)
        rc = self.L.orc_generate_sizes(F, mean, sigma, total is not None, total or 0.0, seed,
                                       int(sigma_relative), _ptr(out, f64p))
        if rc:
            raise ValueError(self.L.orc_last_error().decode())
        return out

    def _collect(self, h, N, J, F):
        streams = []
        for w in range(N):
            p = u32p()
            n = self.L.orc_plan_stream(h, w, C.byref(p))
            streams.append(np.ctypeslib.as_array(p, (n,)).copy() if n else np.empty(0, np.uint32))
        cls = []
        for w in range(N):
            row = []
            for j in range(J):
                p = u32p()
                n = self.L.orc_plan_class_list(h, w, j, C.byref(p))
                row.append(np.ctypeslib.as_array(p, (n,)).copy() if n else np.empty(0, np.uint32))
            cls.append(row)
        po, ph = u64p(), u32p()
        H = self.L.orc_plan_holders(h, C.byref(po), C.byref(ph))
        offs = np.ctypeslib.as_array(po, (F + 1,)).copy()
        hold = (np.ctypeslib.as_array(ph, (H * 3,)).copy().reshape(H, 3) if H
                else np.empty((0, 3), np.uint32))
        self.L.orc_plan_free(h)
        return Plan(N, J, streams, cls, offs, hold)

    def plan(self, seed, F, N, B, E, drop_last, caps, sizes):
        caps = np.ascontiguousarray(caps, np.float64)
        sizes = np.ascontiguousarray(sizes, np.float64)
        h = self.L.orc_plan_build(seed, F, N, B, E, int(drop_last), len(caps),
                                  _ptr(caps, f64p), _ptr(sizes, f64p))
        if not h:
            raise ValueError(self.L.orc_last_error().decode())
        return self._collect(h, N, len(caps), F)

    def assign_from_streams(self, streams, counts, caps, sizes):
        N, F = counts.shape
        ent = np.ascontiguousarray(np.concatenate(streams) if streams else [], np.uint32)
        offs = np.zeros(N + 1, np.uint64)
        offs[1:] = np.cumsum([len(s) for s in streams])
        counts = np.ascontiguousarray(counts, np.uint32)
        caps = np.ascontiguousarray(caps, np.float64)
        sizes = np.ascontiguousarray(sizes, np.float64)
        h = self.L.orc_assign_from_streams(N, F, _ptr(ent, u32p), _ptr(offs, u64p),
                                           _ptr(counts, u32p), len(caps), _ptr(caps, f64p),
                                           _ptr(sizes, f64p))
        return self._collect(h, N, len(caps), F)


class Ref:
    def __init__(self):
        ensure_built(ref=True)
        if not os.path.exists(REF_SO):
            raise FileNotFoundError(REF_SO)
        L = C.CDLL(REF_SO)
        L.ref_last_error.restype = C.c_char_p
        L.ref_rng_stream.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, u64p]
        L.ref_rng_bounded.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, u64p, u64p]
        L.ref_epoch_permutation.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32, u32p]
        L.ref_batch_slice.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32, u64p, u64p]
        L.ref_partition_validate.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32,
                                             C.c_int]
        L.ref_generate_sizes.argtypes = [C.c_uint64, C.c_double, C.c_double, C.c_int, C.c_double,
                                         C.c_uint64, C.c_int, f64p, f64p]
        L.ref_plan_build.restype = C.c_void_p
        L.ref_plan_build.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32,
                                     C.c_int, C.c_uint32, f64p, f64p, C.c_int, C.c_int]
        L.ref_plan_build_subset.restype = C.c_void_p
        L.ref_plan_build_subset.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32,
                                            C.c_uint32, C.c_int, C.c_uint32, f64p, f64p, C.c_int,
                                            u32p, C.c_uint32]
        L.ref_last_phase_ms.argtypes = [f64p]
        L.ref_monte_carlo_histogram.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32, u64p]
        L.ref_expected_hot_samples.restype = C.c_double
        L.ref_expected_hot_samples.argtypes = [C.c_uint32, C.c_uint32, C.c_uint64, C.c_double]
        L.ref_hot_count_threshold.restype = C.c_uint32
        L.ref_hot_count_threshold.argtypes = [C.c_uint32, C.c_uint32, C.c_double]
        L.ref_lemma1_bounds.argtypes = [C.c_uint32, C.c_uint32, C.c_double, C.POINTER(C.c_int64)]
        L.ref_unit_times.argtypes = [C.c_uint32, C.c_uint32, f64p, C.c_uint32, f64p, f64p, f64p]
        L.ref_choose_sources.argtypes = [C.c_void_p, C.c_uint32, C.c_uint32, f64p, u64p, C.c_uint32,
                                         C.c_int, C.c_int, C.c_int, C.c_uint64, u32p, u32p, u32p]
        L.ref_plan_build_subset_lowmem.restype = C.c_void_p
        L.ref_plan_build_subset_lowmem.argtypes = L.ref_plan_build_subset.argtypes
        L.ref_assign_from_streams.restype = C.c_void_p
        L.ref_assign_from_streams.argtypes = [C.c_uint32, C.c_uint32, u32p, u64p, u32p,
                                              C.c_uint32, f64p, f64p]
        for fn in ("ref_plan_stream", "ref_plan_class_list"):
            getattr(L, fn).restype = C.c_uint64
        L.ref_plan_stream.argtypes = [C.c_void_p, C.c_uint32, C.POINTER(u32p)]
        L.ref_plan_epoch_offsets.restype = C.c_uint64
        L.ref_plan_epoch_offsets.argtypes = [C.c_void_p, C.c_uint32, C.POINTER(u64p)]
        L.ref_plan_batch_offsets.restype = C.c_uint64
        L.ref_plan_batch_offsets.argtypes = [C.c_void_p, C.c_uint32, C.POINTER(u64p)]
        L.ref_plan_class_list.argtypes = [C.c_void_p, C.c_uint32, C.c_uint32, C.POINTER(u32p)]
        L.ref_plan_holders.restype = C.c_uint64
        L.ref_plan_holders.argtypes = [C.c_void_p, C.POINTER(u32p), C.POINTER(u32p)]
        L.ref_access_frequencies.argtypes = [C.c_void_p, C.c_uint32, C.c_uint32, C.c_uint32, u32p]
        L.ref_worker_access_counts.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32,
                                               C.c_uint32, C.c_int, C.c_uint32, u32p]
        L.ref_all_access_counts.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32,
                                            C.c_uint32, C.c_int, u32p]
        L.ref_plan_free.argtypes = [C.c_void_p]
        self.L = L

    def err(self):
        return self.L.ref_last_error().decode()

    def rng_stream(self, seed, tag, start, n):
        out = np.empty(n, np.uint64)
        self.L.ref_rng_stream(seed, tag, start, n, _ptr(out, u64p))
        return out

    def epoch_permutation(self, seed, epoch, F):
        out = np.empty(max(F, 1), np.uint32)
        if self.L.ref_epoch_permutation(seed, epoch, F, _ptr(out, u32p)):
            raise ValueError(self.err())
        return out[:F]

    def batch_slice(self, bs, N, w):
        b, e = C.c_uint64(), C.c_uint64()
        self.L.ref_batch_slice(bs, N, w, C.byref(b), C.byref(e))
        return b.value, e.value

    def validate(self, F, N, B, E, drop_last=True):
        if self.L.ref_partition_validate(F, N, B, E, int(drop_last)):
            raise ValueError(self.err())

    def generate_sizes(self, F, mean, sigma, total=None, seed=1, sigma_relative=False):
        out = np.empty(F, np.float64)
        t = C.c_double()
        if self.L.ref_generate_sizes(F, mean, sigma, total is not None, total or 0.0, seed,
                                     int(sigma_relative), _ptr(out, f64p), C.byref(t)):
            raise ValueError(self.err())
        return out

    def _collect(self, h, N, J, F, keep=False):
        streams, eoffs, boffs = [], [], []
        for w in range(N):
            p = u32p()
            n = self.L.ref_plan_stream(h, w, C.byref(p))
            streams.append(np.ctypeslib.as_array(p, (n,)).copy() if n else np.empty(0, np.uint32))
            q = u64p()
            n = self.L.ref_plan_epoch_offsets(h, w, C.byref(q))
            eoffs.append(np.ctypeslib.as_array(q, (n,)).copy())
            n = self.L.ref_plan_batch_offsets(h, w, C.byref(q))
            boffs.append(np.ctypeslib.as_array(q, (n,)).copy())
        cls = []
        for w in range(N):
            row = []
            for j in range(J):
                p = u32p()
                n = self.L.ref_plan_class_list(h, w, j, C.byref(p))
                row.append(np.ctypeslib.as_array(p, (n,)).copy() if n else np.empty(0, np.uint32))
            cls.append(row)
        po, ph = u32p(), u32p()
        H = self.L.ref_plan_holders(h, C.byref(po), C.byref(ph))
        offs = (np.ctypeslib.as_array(po, (F + 1,)).astype(np.uint64) if bool(po)
                else np.zeros(F + 1, np.uint64))
        hold = (np.ctypeslib.as_array(ph, (H * 3,)).copy().reshape(H, 3) if H
                else np.empty((0, 3), np.uint32))
        plan = Plan(N, J, streams, cls, offs, hold)
        plan.epoch_offsets, plan.batch_offsets = eoffs, boffs
        if keep:
            plan._h = h
        else:
            self.L.ref_plan_free(h)
        return plan

    def plan(self, seed, F, N, B, E, drop_last, caps, sizes, mode=0, threads=1, keep=False):
        caps = np.ascontiguousarray(caps, np.float64)
        sizes = np.ascontiguousarray(sizes, np.float64)
        h = self.L.ref_plan_build(seed, F, N, B, E, int(drop_last), len(caps), _ptr(caps, f64p),
                                  _ptr(sizes, f64p), mode, threads)
        if not h:
            raise ValueError(self.err())
        return self._collect(h, N, len(caps), F, keep)

    def plan_subset(self, seed, F, N, B, E, drop_last, caps, sizes, workers, threads):
        caps = np.ascontiguousarray(caps, np.float64)
        sizes = np.ascontiguousarray(sizes, np.float64)
        ws = np.ascontiguousarray(workers, np.uint32)
        h = self.L.ref_plan_build_subset(seed, F, N, B, E, int(drop_last), len(caps),
                                         _ptr(caps, f64p), _ptr(sizes, f64p), threads,
                                         _ptr(ws, u32p), len(ws))
        if not h:
            raise ValueError(self.err())
        return self._collect(h, N, len(caps), F)

    def time_subset(self, seed, F, N, B, E, drop_last, caps, sizes, workers, threads):
        """Builds the per-worker reference plan of a worker subset (every permutation, every
        worker's stream, the subset's assignment, build_index) without copying it out; returns
        the wall-clock phases in ms: permutations, streams, assignment, build_index."""
        caps = np.ascontiguousarray(caps, np.float64)
        sizes = np.ascontiguousarray(sizes, np.float64)
        ws = np.ascontiguousarray(workers, np.uint32)
        h = self.L.ref_plan_build_subset(seed, F, N, B, E, int(drop_last), len(caps),
                                         _ptr(caps, f64p), _ptr(sizes, f64p), threads,
                                         _ptr(ws, u32p), len(ws))
        if not h:
            raise ValueError(self.err())
        ph = np.zeros(4, np.float64)
        self.L.ref_last_phase_ms(_ptr(ph, f64p))
        self.L.ref_plan_free(h)
        return ph

    def plan_subset_lowmem(self, seed, F, N, B, E, drop_last, caps, sizes, workers, threads):
        """Worker-subset plan that never holds all permutations (config 5)."""
        caps = np.ascontiguousarray(caps, np.float64)
        sizes = np.ascontiguousarray(sizes, np.float64)
        ws = np.ascontiguousarray(workers, np.uint32)
        h = self.L.ref_plan_build_subset_lowmem(seed, F, N, B, E, int(drop_last), len(caps),
                                                _ptr(caps, f64p), _ptr(sizes, f64p), threads,
                                                _ptr(ws, u32p), len(ws))
        if not h:
            raise ValueError(self.err())
        return self._collect(h, N, len(caps), F)

    def access_frequencies(self, plan, w, eb, ee, F):
        out = np.empty(F, np.uint32)
        self.L.ref_access_frequencies(plan._h, w, eb, ee, _ptr(out, u32p))
        return out

    def monte_carlo_histogram(self, seed, N, E, F):
        out = np.zeros(E + 1, np.uint64)
        if self.L.ref_monte_carlo_histogram(seed, N, E, F, _ptr(out, u64p)):
            raise ValueError(self.err())
        return out

    def expected_hot_samples(self, N, E, F, delta):
        return self.L.ref_expected_hot_samples(N, E, F, delta)

    def hot_count_threshold(self, N, E, delta):
        return self.L.ref_hot_count_threshold(N, E, delta)

    def lemma1_bounds(self, N, E, delta):
        out = (C.c_int64 * 4)()
        if self.L.ref_lemma1_bounds(N, E, delta, out):
            raise ValueError(self.err())
        return tuple(int(x) for x in out)

    def unit_times(self, N, caps, gamma):
        """fetch_time_local / _remote per class and fetch_time_pfs at size 1.0 on the preset
        reference system (scenarios.cpp:15-46) with these class capacities."""
        caps = np.ascontiguousarray(caps, np.float64)
        J = len(caps)
        lt, rt, pf = np.zeros(max(J, 1)), np.zeros(max(J, 1)), C.c_double()
        if self.L.ref_unit_times(N, J, _ptr(caps, f64p), gamma, _ptr(lt, f64p), _ptr(rt, f64p),
                                 C.byref(pf)):
            raise ValueError(self.err())
        return lt[:J], rt[:J], pf.value

    def choose_sources(self, plan, N, caps, progress, gamma, samples, workers, allow_local=True,
                       allow_remote=True, heuristic=False):
        """The reference's choose_source per query: [n, 3] = (kind, class, worker)."""
        caps = np.ascontiguousarray(caps, np.float64)
        progress = np.ascontiguousarray(progress, np.uint64)
        samples = np.ascontiguousarray(samples, np.uint32)
        workers = np.ascontiguousarray(workers, np.uint32)
        out = np.zeros((len(samples), 3), np.uint32)
        if self.L.ref_choose_sources(plan._h, N, len(caps), _ptr(caps, f64p), _ptr(progress, u64p),
                                     gamma, int(allow_local), int(allow_remote), int(heuristic),
                                     len(samples), _ptr(samples, u32p), _ptr(workers, u32p),
                                     _ptr(out, u32p)):
            raise ValueError(self.err())
        return out

    def free(self, plan):
        if getattr(plan, "_h", None):
            self.L.ref_plan_free(plan._h)
            plan._h = None

    def worker_access_counts(self, seed, F, N, B, E, drop_last, w):
        out = np.empty(F, np.uint32)
        if self.L.ref_worker_access_counts(seed, F, N, B, E, int(drop_last), w, _ptr(out, u32p)):
            raise ValueError(self.err())
        return out

    def all_access_counts(self, seed, F, N, B, E, drop_last):
        out = np.empty((N, F), np.uint32)
        if self.L.ref_all_access_counts(seed, F, N, B, E, int(drop_last), _ptr(out, u32p)):
            raise ValueError(self.err())
        return out

    def assign_from_streams(self, streams, counts, caps, sizes):
        N, F = counts.shape
        ent = np.ascontiguousarray(np.concatenate(streams) if streams else [], np.uint32)
        offs = np.zeros(N + 1, np.uint64)
        offs[1:] = np.cumsum([len(s) for s in streams])
        counts = np.ascontiguousarray(counts, np.uint32)
        caps = np.ascontiguousarray(caps, np.float64)
        sizes = np.ascontiguousarray(sizes, np.float64)
        h = self.L.ref_assign_from_streams(N, F, _ptr(ent, u32p), _ptr(offs, u64p),
                                           _ptr(counts, u32p), len(caps), _ptr(caps, f64p),
                                           _ptr(sizes, f64p))
        if not h:
            raise ValueError(self.err())
        return self._collect(h, N, len(caps), F)


def plans_equal(a: Plan, b: Plan, check_streams=True) -> str | None:
    """Return None when bit-identical, else a description of the first difference."""
    if a.N != b.N or a.J != b.J:
        return "shape"
    if check_streams:
        for w in range(a.N):
            if not np.array_equal(a.streams[w], b.streams[w]):
                return f"stream of worker {w}"
    for w in range(a.N):
        for j in range(a.J):
            if not np.array_equal(a.class_lists[w][j], b.class_lists[w][j]):
                return f"class list worker {w} class {j + 1}"
    if not np.array_equal(a.holder_offsets.astype(np.uint64), b.holder_offsets.astype(np.uint64)):
        return "holder offsets"
    if not np.array_equal(a.holders, b.holders):
        return "holders"
    return None
