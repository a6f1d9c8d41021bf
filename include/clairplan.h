/* clairplan — B200-native NoPFS clairvoyant plan build, C ABI (the drop-in boundary).
 *
 * The reference (clairsim, /root/reference/proj) exposes this path as C++ free functions in
 * namespace clairsim with host std::vector results.  Each entry point below names the
 * reference interface it replaces (path:line, relative to /root/reference/proj).  The
 * C++ shim paper_2101_08734_b200/csrc/compat/clairsim_compat.cpp re-exports the exact
 * clairsim:: signatures on top of these calls; INTEGRATION.md shows the bindings.
 *
 * Conventions
 *  - Every call returns an int status: CLAIRPLAN_OK (0) or one of the codes below; the
 *    message for the calling thread is clairplan_last_error().  Validation failures use
 *    the reference's exact std::invalid_argument texts (access.cpp:41-50, :53).
 *  - Plain pointers and sizes only; "host" buffers are caller-owned CPU memory, "device"
 *    buffers live on the handle's CUDA device and stay owned by the handle.
 *  - Handles are independent (own CUDA stream + workspace): concurrent calls on different
 *    handles from different host threads are safe, as the reference's sweep pool requires
 *    (simulator.cpp:471-480).  One handle must not be used by two threads at once.
 *  - There is no CPU fallback: without a usable sm_100 device every compute call returns
 *    CLAIRPLAN_ENODEV.
 */
#ifndef CLAIRPLAN_H
#define CLAIRPLAN_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CLAIRPLAN_OK 0
#define CLAIRPLAN_ENOMEM 12    /* device or host allocation failed */
#define CLAIRPLAN_ENODEV 19    /* no CUDA device / not sm_100 */
#define CLAIRPLAN_EINVAL 22    /* invalid argument (reference message text) */
#define CLAIRPLAN_ERANGE 34    /* caller buffer too small */
#define CLAIRPLAN_EOVERFLOW 75 /* result does not fit the requested (reference u32) layout */
#define CLAIRPLAN_ECUDA 1001   /* CUDA runtime error */
#define CLAIRPLAN_ENCCL 1002   /* NCCL error (multi-GPU) */

typedef struct clairplan_plan* clairplan_t;

/* Everything nopfs_assign_caches + build_access_streams read (policies.cpp:144-166,
 * access.cpp:59-78): Seed, PartitionSpec, SystemConfig::storage[1..J].capacity_mb and
 * DatasetModel::sizes_mb. */
typedef struct {
    uint64_t seed;              /* Seed::value                        access.hpp:14-16 */
    uint32_t samples;           /* F = DatasetModel::samples           perfmodel.hpp:60 */
    uint32_t num_workers;       /* PartitionSpec::num_workers          access.hpp:20 */
    uint32_t global_batch;      /* PartitionSpec::global_batch (B)     access.hpp:21 */
    uint32_t epochs;            /* PartitionSpec::epochs               access.hpp:22 */
    int32_t drop_last;          /* PartitionSpec::drop_last            access.hpp:23 */
    uint32_t num_classes;       /* J = SystemConfig::cache_class_count perfmodel.hpp:55 */
    const double* capacities_mb; /* host [J]: storage[1..J].capacity_mb */
    const double* sizes_mb;     /* [F] DatasetModel::sizes_mb, host or device */
    int32_t sizes_on_device;    /* 1: sizes_mb is a device pointer on `device` */
    int32_t device;             /* CUDA ordinal */
    uint32_t worker_begin;      /* worker range planned by this handle: [begin, end); */
    uint32_t worker_end;        /*   0,0 = all workers (single-GPU plan) */
} clairplan_config;

/* Per-build counters. */
typedef struct {
    uint64_t accesses;        /* A: stream entries of the handle's workers */
    uint64_t pairs;           /* D: distinct (worker, sample) pairs of those workers */
    uint64_t holders;         /* assigned pairs = holder records */
    uint64_t rejections;      /* Lemire rejections resolved (rng.hpp:54-60) */
    double device_ms;         /* device time of the last clairplan_build (CUDA events) */
    uint32_t path;            /* pipeline of the last build: CLAIRPLAN_PATH_* */
    uint32_t reserved;
} clairplan_stats;

#define CLAIRPLAN_PATH_V1 0      /* generic / v1 pipeline (explicit streams, large handles) */
#define CLAIRPLAN_PATH_TIER 1    /* v2: tier order + exact first fit */
#define CLAIRPLAN_PATH_ALLFIT 2  /* v2: every worker provably fits class 1 (no tier order) */

int clairplan_version(void);
const char* clairplan_last_error(void);

/* PartitionSpec::validate (access.cpp:41-50) with the same messages. */
int clairplan_validate(const clairplan_config* cfg);

/* Allocates the handle, its stream and workspace; copies capacities and sizes. */
int clairplan_create(const clairplan_config* cfg, clairplan_t* out);
int clairplan_destroy(clairplan_t plan);

/* The whole hot path, device-resident: epoch permutations -> per-worker streams ->
 * (count, first-access) per (worker, sample) -> tier assignment -> prefetch orders ->
 * holder CSR.  Replaces build_access_streams (access.cpp:59-78) + access_frequencies for
 * every worker + nopfs_assign_caches + build_index (policies.cpp:446-456).  Synchronous. */
int clairplan_build(clairplan_t plan);
int clairplan_stats_get(clairplan_t plan, clairplan_stats* out);

/* ---- device views (valid until the next build/destroy) ---------------------------- */
/* Worker-major streams: worker w's AccessStream::entries (access.hpp:32-43) is
 * entries[stream_offset(w) .. stream_offset(w+1)). */
int clairplan_device_streams(clairplan_t plan, const uint32_t** entries, uint64_t* total);
uint64_t clairplan_stream_offset(clairplan_t plan, uint32_t worker);
/* CacheAssignment::class_lists[w][j-1] (policies.hpp:56-57), prefetch-ordered:
 * entries[off[w*J + j-1] .. off[w*J + j-1] + len[w*J + j-1]) — host arrays filled here. */
int clairplan_class_list_bounds(clairplan_t plan, uint64_t* off, uint64_t* len);
int clairplan_device_class_lists(clairplan_t plan, const uint32_t** entries);
/* CacheAssignment::holder_offsets/holders (policies.hpp:58-61) with u64 offsets:
 * offsets[F+1], holders = {worker, storage_class (1-based), position} x count. */
int clairplan_device_holders(clairplan_t plan, const uint64_t** offsets,
                             const uint32_t** holders, uint64_t* count);

/* ---- host export ------------------------------------------------------------------- */
int clairplan_export_stream(clairplan_t plan, uint32_t worker, uint32_t* out, uint64_t cap,
                            uint64_t* len);
int clairplan_export_streams(clairplan_t plan, uint32_t* out, uint64_t cap);
/* all class lists, (w, j)-major, with the N*J bounds from clairplan_class_list_bounds */
int clairplan_export_class_lists(clairplan_t plan, uint32_t* out, uint64_t cap);
int clairplan_export_holders(clairplan_t plan, uint64_t* offsets, uint32_t* holders,
                             uint64_t cap);
/* FrequencyTable::counts of worker w over all epochs (access.cpp:80-88), dense [F]. */
int clairplan_export_counts(clairplan_t plan, uint32_t worker, uint32_t* counts);

/* ---- stand-alone entry points of the same path --------------------------------------- */
/* epoch_permutation (access.hpp:58, access.cpp:52-57) into a host buffer [samples]. */
int clairplan_epoch_permutation(uint64_t seed, uint32_t epoch, uint32_t samples,
                                uint32_t* out, int device);
/* access_frequencies (access.hpp:66-67): entries/epoch_offsets are one host AccessStream. */
int clairplan_access_frequencies(const uint32_t* entries, const uint64_t* epoch_offsets,
                                 uint32_t epoch_count, uint32_t samples, uint32_t epoch_begin,
                                 uint32_t epoch_end, uint32_t* counts, int device);
/* worker_access_counts / all_access_counts (access.hpp:71-77); all: counts is [N][F]. */
int clairplan_worker_access_counts(const clairplan_config* cfg, uint32_t worker,
                                   uint32_t* counts);
int clairplan_all_access_counts(const clairplan_config* cfg, uint32_t* counts);
/* nopfs_assign_caches (policies.hpp:88-90) on caller-supplied streams and dense
 * frequency tables (N x F).  Creates a handle whose class lists / holders are readable
 * through the calls above.  entries: concatenated streams, offsets[N+1]. */
int clairplan_assign_from_streams(uint32_t num_workers, uint32_t samples,
                                  const uint32_t* entries, const uint64_t* offsets,
                                  const uint32_t* counts, uint32_t num_classes,
                                  const double* capacities_mb, const double* sizes_mb,
                                  int device, clairplan_t* out);

/* CacheAssignment::build_index (policies.cpp:124-142) for caller-edited class lists:
 * entries = class lists concatenated in (worker, class) order, list_off[N*J + 1];
 * offsets_out[samples+1] (u64) and holders_out[3 x total] in build_index order. */
int clairplan_build_index(uint32_t num_workers, uint32_t num_classes, uint64_t samples,
                          const uint32_t* entries, const uint64_t* list_off,
                          uint64_t* offsets_out, uint32_t* holders_out, int device);

/* Re-planning (capacity sweeps): new storage[1..J].capacity_mb for a built handle; reruns
 * first fit, prefetch orders and holders on the cached streams/tables (simulator.cpp:457-465
 * rebuilds everything per grid point). */
int clairplan_reassign(clairplan_t plan, const double* capacities_mb);

/* ---- multi-GPU building blocks (one process per GPU, NCCL between the calls) ---------- */
/* Permutation rows of epochs [epoch_begin, epoch_begin+count) into a device buffer
 * d_out[count][F] (epoch_permutation for each epoch, rejections resolved). */
int clairplan_generate_perms(clairplan_t plan, uint32_t epoch_begin, uint32_t epoch_count,
                             uint32_t* d_out);
/* clairplan_build for the handle's worker range from all E permutation rows d_perms[E][F]
 * (e.g. epoch-sharded rows all-gathered over NVLink). */
int clairplan_build_from_perms(clairplan_t plan, const uint32_t* d_perms);
/* Epoch-range streams (the all-to-all exchange of the sharded build): the streams of ALL
 * workers for epochs [epoch_begin, epoch_begin+count), laid out worker-major as
 * build_access_streams would for a run of `count` epochs (access.cpp:59-78):
 * d_out[prefix(w)*count + (e-epoch_begin)*len(w) + t]; the range for the workers of rank d
 * is contiguous, [count*prefix(wb_d), count*prefix(we_d)), prefix = clairplan_epoch_prefix.
 * Rejections resolved.  Replaces epoch_permutation x count (access.cpp:52-57). */
int clairplan_generate_streams(clairplan_t plan, uint32_t epoch_begin, uint32_t epoch_count,
                               uint32_t* d_out);
/* Stream entries per epoch of the workers below `worker` (sum of batch_slice lengths). */
int clairplan_epoch_prefix(clairplan_t plan, uint32_t worker, uint64_t* entries);
/* clairplan_build for the handle's worker range from the all-to-all output d_recv: for each
 * source rank r (epochs [epoch_bounds[r], epoch_bounds[r+1])) its block
 * [local worker][epoch][t], blocks in rank order.  epoch_bounds[nsrc+1] is host memory. */
int clairplan_build_from_streams(clairplan_t plan, const uint32_t* d_recv,
                                 const uint32_t* epoch_bounds, uint32_t nsrc);
/* Fused exchange (multi-GPU on one node, CUDA IPC peer memory over NVLink/NVSwitch): the
 * epoch-range shuffle writes every stream entry straight into the receive buffer of the rank
 * owning its worker, replacing generate_streams + the all-to-all.  Rank d (workers
 * [worker_bounds[d], worker_bounds[d+1])) receives entry idx of this rank's epoch-range
 * stream layout at ((uint32_t*)dst_base[d])[idx + dst_delta[d]], i.e. the receive layout of
 * clairplan_build_from_streams.  The caller orders the ranks (a barrier after this call,
 * before the owners build; receive buffers not reused while an owner still reads them).
 * Bucketed shuffle only (clairplan_p2p_supported). */
int clairplan_generate_streams_p2p(clairplan_t plan, uint32_t epoch_begin, uint32_t epoch_count,
                                   const uint64_t* dst_base, const int64_t* dst_delta,
                                   const uint32_t* worker_bounds, uint32_t nranks);
int clairplan_p2p_supported(clairplan_t plan);
/* Receive buffer i (< 4) of the handle's local entries (allocated on first use, freed with the
 * handle) and its CUDA IPC handle (64 bytes, may be NULL); peers open it with
 * clairplan_open_peer_buffer (closed with the handle). */
int clairplan_recv_buffer(clairplan_t plan, uint32_t i, void** d_ptr, void* ipc_handle);
int clairplan_open_peer_buffer(clairplan_t plan, const void* ipc_handle, void** d_ptr);
/* Per-sample number of holder records of the handle's workers, d_out[F] (device): the
 * input of the cross-GPU holder-offset merge (all-gather + exclusive scan over ranks). */
int clairplan_holder_counts(clairplan_t plan, uint32_t* d_out);
/* Holder-offset merge of a worker-sharded plan on `stream` (0: the legacy default stream): d_allc =
 * [world][F] per-rank per-sample holder counts (the all-gather of clairplan_holder_counts),
 * d_glob[F + 1] = global CSR offsets, d_starts[F] = where this rank's records of each sample
 * start (ranks own ascending worker ranges: build_index's order, policies.cpp:124-142). */
int clairplan_merge_holder_counts(clairplan_t plan, const uint32_t* d_allc, uint32_t world,
                                  uint32_t rank, int64_t* d_glob, int64_t* d_starts, void* stream);
/* Overlap of that merge with the build's tail (no reference counterpart: the reference is a
 * single process).  During the next builds, as soon as the per-sample pair counts exist,
 * they are copied into d_counts[F] (device), `stream` (a cudaStream_t, e.g. the caller's
 * collective stream) is made to wait for the copy and fn(user) runs on the calling thread —
 * once per build, on every rank at the same point — to enqueue the all-gather.  fn = NULL
 * removes the hook. */
int clairplan_set_counts_hook(clairplan_t plan, uint32_t* d_counts, void* stream,
                              void (*fn)(void*), void* user);
/* 1 if the last build's hooked counts are its holder counts (all-fit path: every pair is a
 * holder; no rejection rerun after the hook), else 0: merge again from
 * clairplan_holder_counts. */
int clairplan_counts_hook_valid(clairplan_t plan);

/* Host-side input generator: DatasetModel::generate (perfmodel.cpp:68-99), bit-identical
 * with the reference built with the same glibc (no FMA contraction).  Not timed. */
int clairplan_generate_sizes(uint64_t samples, double mean_mb, double sigma_mb, int has_total,
                             double total_mb, uint64_t seed, int sigma_relative, double* out);

/* Number of kernel launches issued by the last clairplan_build on this handle. */
uint64_t clairplan_launch_count(clairplan_t plan);
/* Device time per pipeline stage of the last build (CUDA events on the handle's stream);
 * returns the number of stages; names via clairplan_stage_name. */
int clairplan_stage_times(clairplan_t plan, double* ms, uint32_t n);
const char* clairplan_stage_name(uint32_t stage);
/* End to end in one call (the reference's build_policy returns host vectors,
 * policies.cpp:446-456): sizes from host memory (optional, NULL keeps the handle's), the
 * build, and every output copied to host buffers — streams (layout of
 * clairplan_export_streams), class lists (clairplan_export_class_lists), holder CSR
 * (clairplan_export_holders).  The stream copy starts as soon as the streams are final and
 * overlaps the rest of the build on a second CUDA stream; pinned buffers make it asynchronous. */
int clairplan_build_export(clairplan_t plan, const double* host_sizes, uint32_t* streams_out,
                           uint64_t streams_cap, uint32_t* class_lists_out, uint64_t cl_cap,
                           uint64_t* offsets_out, uint32_t* holders_out, uint64_t holders_cap);
/* Replaces the sample sizes (DatasetModel::sizes_mb) of a handle, e.g. from pinned host
 * memory for an end-to-end step; the copy is ordered before the next build. */
int clairplan_set_sizes(clairplan_t plan, const double* sizes_mb, int on_device);

/* ---- plan consumer ----------------------------------------
 * Replaces per-access calls of nopfs_choose_source / choose_source / best_cached_source
 * (policies.hpp:100-117, policies.cpp:168-233) with one batched device call over the plan's
 * holder CSR.  Kinds follow FetchSource::Kind (policies.hpp:77-82). */
#define CLAIRPLAN_SRC_PFS 0
#define CLAIRPLAN_SRC_REMOTE 1
#define CLAIRPLAN_SRC_LOCAL 2
typedef struct {
    uint8_t kind;           /* CLAIRPLAN_SRC_* */
    uint8_t storage_class;  /* 1-based (Remote / Local), 0 for the PFS */
    uint16_t reserved;
    uint32_t worker;        /* holder (Remote), the requester (Local), 0 (PFS) */
} clairplan_source;
/* n queries (samples[i], workers[i]); progress[w * J + j] = PrefetchProgress::completed[w][j]
 * for ALL N workers (u64, policies.hpp:73-75); local_time / remote_time[j] = fetch_time_local /
 * fetch_time_remote(1.0, cfg, j + 1), pfs_time = fetch_time_pfs(1.0, cfg, gamma)
 * (perfmodel.cpp:109-121); on_device: every pointer but the two time tables is device memory.
 * nopfs_choose_source = allow_local = allow_remote = 1. */
int clairplan_choose_sources(clairplan_t plan, uint64_t n, const uint32_t* samples,
                             const uint32_t* workers, const uint64_t* progress,
                             const double* local_time, const double* remote_time, double pfs_time,
                             int allow_local, int allow_remote, int heuristic, int on_device,
                             clairplan_source* out);
/* "Earliest remote holder" table: per sample, out[3k..3k+2] = {worker, class, position} of
 * the holder with the smallest (remote_time[class-1], position, worker); all 0xFFFFFFFF for
 * samples nobody caches.  A derived view (the reference scans holders_of per access). */
int clairplan_earliest_holders(clairplan_t plan, const double* remote_time, uint32_t* out);

/* ---- analysis reuse: counts stay on the device ------------------------
 * FrequencyHistogram of one worker's counts on a built plan: buckets[c] = samples the worker
 * accesses exactly c times (c > max_count lands in buckets[max_count]); analysis.hpp:33-41. */
int clairplan_count_histogram(clairplan_t plan, uint32_t worker, uint32_t max_count,
                              uint64_t* buckets);
/* monte_carlo_histogram (analysis.cpp:84-96): worker 0 of the B = N, drop_last = false
 * partition; buckets[0..epochs]. */
int clairplan_monte_carlo_histogram(uint64_t seed, uint32_t workers, uint32_t epochs,
                                    uint32_t samples, uint64_t* buckets, int device);
/* Per sample the largest / smallest access count over all workers (the inputs of the Lemma-1
 * property suite, acceptance.cpp:98-158), from the device counts. */
int clairplan_count_extremes(const clairplan_config* cfg, uint32_t* hi, uint32_t* lo);

/* ---- plan wire format -------------------------------------------------
 * A versioned binary image of one handle's plan for files and for distribution (the paper's
 * middleware all-gathers the access information at setup; the reference
 * has no serialization).  Sections follow the header at the recorded offsets (16-B aligned):
 * capacities f64[J], streams u32[A], class bounds u64[2 * nloc * J] ({offset, length} into
 * the class-list section, worker-major), class lists u32[class_entries], holder offsets
 * u64[F + 1], holders u32[3 * holders].  checksum[s] = sum_i mix64((s << 56) + i * golden)
 * ^ word_i (mod 2^64) over the 32-bit words of section s (0 caps .. 5 holders). */
#define CLAIRPLAN_WIRE_VERSION 1
typedef struct {
    char magic[8];              /* "CLPLAN\0\1" */
    uint32_t version, header_bytes;
    uint64_t seed;
    uint32_t samples, num_workers, global_batch, epochs;
    uint32_t drop_last, num_classes, worker_begin, worker_end;
    uint64_t accesses, class_entries, holders;
    uint64_t off_caps, off_streams, off_class_bounds, off_class_lists, off_holder_offsets,
        off_holders, total_bytes;
    uint64_t checksum[6];
    uint8_t reserved[256 - 8 - 8 - 8 - 32 - 24 - 56 - 48];
} clairplan_wire_header;
int clairplan_wire_size(clairplan_t plan, uint64_t* bytes);
int clairplan_wire_write(clairplan_t plan, void* out, uint64_t cap);
/* Section checksums of the image this handle contributes to a merged (all-shard) image,
 * computed on the device without any copy: the streams start at word stream_base of the
 * merged streams section, the class lists at entry list_base, and the holder records at the
 * global CSR positions d_holder_starts[k] + local rank (device u64[F]; null: the handle's own
 * CSR, whose offsets are then summed too).  out[1] streams, out[3] class lists, out[4] holder
 * offsets (own CSR only), out[5] holders; out[0], out[2] are 0.  Summing the shards' values
 * (mod 2^64) gives the merged image's checksums: a scale-free cross-check of sharded builds. */
int clairplan_wire_checksums(clairplan_t plan, uint64_t stream_base, uint64_t list_base,
                             const uint64_t* d_holder_starts, uint64_t* out);

#ifdef __cplusplus
}
#endif
#endif /* CLAIRPLAN_H */
