// Internal declarations shared by the clairplan translation units (not part of the ABI).
#pragma once
#include <cuda_runtime.h>

#include <algorithm>
#include <stddef.h>
#include <stdint.h>
#include <vector>

#include "common.cuh"

namespace clairplan {

// Bump allocator over one device buffer; all users run on one stream, so memory released
// by mark/release may be reused by later kernels of the same stream.
struct Workspace {
    char* base = nullptr;
    size_t cap = 0, used = 0, peak = 0;
    bool overflow = false;
    template <typename T>
    T* scratch(uint64_t n) {
        const size_t bytes = ((size_t)n * sizeof(T) + 255) & ~(size_t)255;
        if (used + bytes > cap) {
            overflow = true;
            return nullptr;
        }
        T* p = reinterpret_cast<T*>(base + used);
        used += bytes;
        if (used > peak) peak = used;
        return p;
    }
    size_t mark() const { return used; }
    void release(size_t m) { used = m; }
};

// Tiles of `tile` elements over segments (never straddling one).
struct TileMap {
    uint32_t tile = 0, nseg = 0;
    uint64_t max_tiles = 0;        // upper bound; tile_seg[t] == kNone past the real count
    uint64_t* tile_base = nullptr; // [nseg+1] first tile of each segment
    uint32_t* tile_seg = nullptr;  // [max_tiles]
};

// per local worker: sum / count of its candidates' sizes (all-fit test); sum == nullptr: off
// exact 64-bit add into a (lo, hi) pair of shared words with 32-bit atomics (shared 64-bit
// atomic adds compile to CAS loops)
__device__ __forceinline__ void add64(uint32_t* lo, uint32_t* hi, unsigned long long v) {
    const uint32_t vl = (uint32_t)v, vh = (uint32_t)(v >> 32);
    const uint32_t old = atomicAdd(lo, vl);
    const uint32_t carry = (uint32_t)(old + vl < old);
    if (vh + carry) atomicAdd(hi, vh + carry);
}

struct WorkerSums {
    const double* sizes = nullptr;
    unsigned long long* sum = nullptr;  // sum of ceil(size * 2^20): an upper bound
    uint32_t* cnt = nullptr;
    uint32_t* neg = nullptr;  // set when a size is negative (or NaN)
};

void exclusive_scan(cudaStream_t s, const uint32_t* in, uint64_t n, uint64_t* out, Workspace& ws);
void exclusive_scan(cudaStream_t s, const uint64_t* in, uint64_t n, uint64_t* out, Workspace& ws);

void build_tilemap(cudaStream_t s, const uint64_t* seg_len, uint32_t nseg, uint64_t total_len,
                   uint32_t tile, TileMap& tm, Workspace& ws);
void radix_pass(cudaStream_t s, const TileMap& tm, const uint64_t* seg_begin,
                const uint64_t* seg_len, const uint32_t* keys, const uint32_t* vals,
                uint32_t shift, uint32_t* okeys, uint32_t* ovals, uint32_t* dest,
                uint64_t** scanned_out, Workspace& ws);
void radix_regions(cudaStream_t s, const TileMap& tm, const uint64_t* seg_begin,
                   const uint64_t* seg_len, const uint64_t* scanned, uint32_t ndig,
                   uint64_t* rstart, uint64_t* rlen);
constexpr uint32_t kRadixTile = 2048;

void launch_fy_link(cudaStream_t s, uint64_t key, uint32_t F, uint32_t e0, uint32_t ne,
                    uint32_t* head, uint32_t* next, const RejTable& rt, uint32_t* rej_flag,
                    bool detect_only, uint32_t i_limit);
// Multi-GPU fused exchange: the shuffle writes every stream entry straight into the receive
// buffer of the rank owning its worker (CUDA IPC peer memory over NVLink) instead of a local
// send buffer + all-to-all.  Entry idx of the local epoch-range stream layout goes to
// base[d][idx + delta[d]] for the rank d with wb[d] <= worker < wb[d+1].
constexpr uint32_t kMaxPeers = 16;
struct StreamDst {
    uint32_t G = 0;  // 0: the local stream buffer
    uint32_t wb[kMaxPeers + 1] = {};
    uint32_t* base[kMaxPeers] = {};
    long long delta[kMaxPeers] = {};
};
// contiguous-bucket Fisher-Yates resolution for large F (perm_fyc.cu)
struct FycHost {
    uint32_t F = 0, NB = 0, lgW = 0, pack = 0;
    uint64_t rtotal = 0;
    std::vector<uint32_t> bstart, cap, cell;  // block starts [NB+1], capacities, target cells
    std::vector<uint64_t> roff;               // region offsets [NB+1]
};
struct FycDev {
    uint32_t NB = 0, lgW = 0, pack = 0;
    uint64_t rtotal = 0;
    const uint32_t* bstart = nullptr;
    const uint32_t* cell = nullptr;
    const uint32_t* roff = nullptr;
    const uint32_t* cap = nullptr;
};
bool fyc_plan(uint32_t F, FycHost& h);
uint32_t fyc_epochs_per_batch(uint32_t F, uint32_t E);
void launch_fyc(cudaStream_t s, uint64_t key, const Part& part, uint32_t e0, uint32_t ne,
                const FycDev& g, const RejTable& rt, uint32_t* rej_flag, uint32_t* region,
                uint32_t* cursor, uint32_t* tsucc, uint32_t* q, uint32_t* inv, uint32_t* stream,
                uint32_t* perm_out, const StreamDst* dst);
constexpr uint32_t kRejOverflow = 0x80000000u;  // rej_flag bit: a fyc block region overflowed

void launch_fy_group(cudaStream_t s, uint32_t F, uint32_t ne, const uint32_t* head,
                     uint32_t* next, uint32_t* q, uint32_t* scratch, uint32_t scratch_cap,
                     uint32_t* scratch_used, uint32_t* err);
void launch_fy_emit(cudaStream_t s, uint64_t key, const Part& part, uint32_t e0, uint32_t ne,
                    const uint32_t* succ, const uint32_t* q, const RejTable& rt, uint32_t* inv,
                    uint32_t* stream, uint32_t* perm_out);

// epoch ranges of the source ranks of an all-to-all: source r holds [eb[r], eb[r+1])
constexpr uint32_t kMaxRanks = 64;
struct EpochSplit {
    uint32_t G;
    uint32_t eb[kMaxRanks + 1];
};
void launch_stream_relayout(cudaStream_t s, const Part& part, const EpochSplit& es,
                            const uint32_t* recv, uint32_t* stream);
bool sparse_path_ok(const Part& part, uint64_t local_entries);
bool sparse_path_fits(const Part& part);
uint64_t csr_windows(uint64_t n);
void launch_sparse_csr(cudaStream_t s, const Part& part, const uint32_t* stream, uint64_t n,
                       uint32_t* cnt, uint64_t* koff, uint32_t* cur, uint32_t* csr, uint32_t* cpos,
                       uint64_t* soff, Workspace& ws);
void launch_sparse_sample(cudaStream_t s, const Part& part, const uint64_t* soff, const uint64_t* koff,
                          const uint32_t* csr, uint32_t* pair_count, uint16_t* einfo,
                          uint16_t* erank, const WorkerSums& ws);
void launch_holder_sparse(cudaStream_t s, const Part& part, uint64_t n, const uint64_t* soff,
                          const uint32_t* stream, const uint32_t* csr, const uint16_t* erank,
                          uint32_t MB, const uint32_t* rec, uint32_t np, uint32_t J, uint32_t Rp,
                          const uint32_t* cbase, const uint64_t* pair_off, uint32_t* holders,
                          bool allfit,
                          const uint32_t* gate = nullptr);
void launch_stream_inv(cudaStream_t s, const Part& part, const uint32_t* stream, uint32_t* inv,
                       uint32_t skip_lo = 0, uint32_t skip_hi = 0);
void launch_perm_scatter(cudaStream_t s, const Part& part, const uint32_t* perms, uint32_t* inv,
                         uint32_t* stream);

int sample_pass_config(const Part& part, uint32_t* hs, uint32_t* nw_words, uint32_t* warps,
                       size_t* smem);
void launch_sample_pass(cudaStream_t s, const Part& part, uint32_t* info, uint32_t* pair_count,
                        uint32_t hs, uint32_t nw_words, uint32_t warps, size_t smem);

void launch_seg_count(cudaStream_t s, const Part& part, const uint32_t* stream,
                      const uint32_t* info, uint32_t* segcnt);
void launch_seg_write(cudaStream_t s, const Part& part, const uint32_t* stream,
                      const uint32_t* info, const uint64_t* seg_off, uint32_t* cand_k,
                      uint32_t* cand_info);
void launch_worker_segments(cudaStream_t s, const uint64_t* seg_off, uint32_t nloc, uint32_t E,
                            uint64_t* wbegin, uint64_t* wlen);

void first_fit_pass(cudaStream_t s, const uint64_t* seg_begin, const uint64_t* seg_len,
                    uint32_t nseg, uint64_t total, const double* sz, double C, uint8_t* taken,
                    Workspace& ws, unsigned long long* taken_count = nullptr,
                    const uint32_t* gather_idx = nullptr, const double* gather_src = nullptr);

void compact_rejects(cudaStream_t s, const uint64_t* seg_begin, const uint64_t* seg_len,
                     uint32_t nseg, uint64_t total, const uint8_t* taken, const uint32_t* seq_idx,
                     const double* sorted_size, uint64_t out0, uint32_t* out_idx, double* out_sz,
                     uint64_t* nb, uint64_t* nl, Workspace& ws);
void launch_gather_sizes(cudaStream_t s, const uint32_t* order, const uint32_t* cand_k,
                         const double* sizes, uint64_t n, double* out);
void launch_count_keys(cudaStream_t s, const uint32_t* cand_info, uint64_t n, uint32_t maxc,
                       uint32_t* keys);
void launch_apply_pass(cudaStream_t s, const uint8_t* taken, uint64_t n,
                       const uint32_t* seq_to_sorted, const uint32_t* order, uint8_t cls,
                       uint8_t* cand_cls);
void launch_reject_keys(cudaStream_t s, const uint8_t* taken, uint64_t n,
                        const uint32_t* seq_to_sorted, uint32_t* keys, uint32_t* vals);
void launch_gather_seq_sizes(cudaStream_t s, const uint32_t* idx, const double* sorted_size,
                             const uint64_t* seg_begin, const uint64_t* seg_len, uint32_t nseg,
                             double* out);
void launch_class_keys(cudaStream_t s, const uint8_t* cand_cls, uint64_t n, uint32_t J,
                       uint32_t* keys);
void launch_holder_scatter(cudaStream_t s, const uint32_t* cand_k, const uint32_t* cand_info,
                           const uint8_t* cand_cls, const uint32_t* dest, const uint64_t* wbegin,
                           const uint64_t* wlen, const uint64_t* class_start, uint32_t J,
                           uint32_t nloc, uint32_t worker0, const uint64_t* pair_off,
                           uint32_t* holders);
void launch_holder_count(cudaStream_t s, const uint64_t* pair_off, uint32_t F, const uint32_t* tmp,
                         uint32_t* cnt);
void launch_holder_compact(cudaStream_t s, const uint64_t* pair_off, uint32_t F,
                           const uint32_t* tmp, const uint64_t* hoff, uint32_t* holders);
void launch_stream_hist(cudaStream_t s, const uint32_t* st, uint64_t n, uint32_t* counts);

// v2 seed path (fastpath.cu)
bool lane_path_ok(const Part& part);
void launch_sample_lanes(cudaStream_t s, const Part& part, const uint32_t* inv, uint16_t* info,
                         uint16_t* rank16, uint32_t* pair_count, uint32_t* seghist);
bool tile_path_ok(const Part& part);
void launch_sample_tile(cudaStream_t s, const Part& part, const uint32_t* inv, void* info, bool info8,
                        uint16_t* rank16, uint32_t* pair_count, uint32_t* seghist,
                        const WorkerSums& ws);
void launch_sample_hash(cudaStream_t s, const Part& part, const uint32_t* inv, uint16_t* info,
                        uint16_t* rank16, uint32_t* pair_count, const uint32_t* list,
                        const uint32_t* nlist, uint64_t max_items, uint32_t* seghist);
void launch_segcnt(cudaStream_t s, uint32_t nloc, uint32_t E, const uint32_t* seghist,
                   uint32_t* segcnt);
void launch_seg_hist(cudaStream_t s, const Part& part, const uint32_t* stream, const void* info,
                     bool info8, const uint32_t* cpos, uint32_t* seghist, uint32_t* segcnt);
constexpr uint32_t kAllfitChunk = 1024;
void launch_seg_allfit(cudaStream_t s, const Part& part, const uint32_t* stream, const void* info,
                       bool info8, const uint32_t* cpos, uint32_t MB, uint32_t C,
                       unsigned long long* status, uint32_t* ticket, uint32_t* rec,
                       uint32_t* class_list, const uint32_t* gate = nullptr);
void launch_allfit_meta(cudaStream_t s, const Part& part, uint32_t J, const uint32_t* wcnt,
                        uint64_t* clen, uint64_t* cstart, uint32_t* cbase,
                        const uint32_t* gate = nullptr);
void launch_allfit_decide(cudaStream_t s, uint32_t nloc, const unsigned long long* wsum,
                          const uint32_t* wcnt, double C, uint32_t* ok);
void launch_seg_write2(cudaStream_t s, const Part& part, const uint32_t* stream, const uint16_t* info, const uint32_t* cpos,
                       const double* sizes, const uint64_t* seg_off, const uint64_t* sorted_base,
                       uint32_t MB, uint32_t* dest, double* sorted_size, uint32_t* blkmask,
                       uint32_t* blkbase);
// tier.cu (dense tier path)
void launch_seg_write3(cudaStream_t s, const Part& part, const uint32_t* stream, const void* info,
                       bool info8, const uint64_t* seg_off, const uint64_t* sorted_base, uint32_t MB,
                       uint32_t* dest, uint32_t* sorted_k, uint32_t* blkmask, uint32_t* blkbase,
                       uint32_t* claim);
void launch_gather_sorted_sizes(cudaStream_t s, const uint32_t* sorted_k, const double* sizes,
                                uint64_t n, double* out);
void launch_fill_class(cudaStream_t s, uint8_t* cls, uint64_t n, uint8_t j);
void launch_hp_fill(cudaStream_t s, const Part& part, const uint32_t* inv, const uint16_t* rank16,
                    uint32_t MB, const uint32_t* rec, uint32_t np, uint32_t J, uint32_t Rp,
                    const uint32_t* cbase, uint32_t* hp, uint32_t* claim);
bool holder_hp_ok(const Part& part);  // E within one TMA box, tiles within shared memory
void launch_holder_hp(cudaStream_t s, const Part& part, const uint32_t* inv, const uint16_t* rank16,
                      const uint32_t* hp, const uint64_t* pair_off, uint32_t* holders);
void launch_blk_codes(cudaStream_t s, const Part& part, uint32_t MB, const uint32_t* blkmask,
                      const uint32_t* blkbase, const uint32_t* dest, const uint8_t* cls_sorted,
                      uint32_t np, uint32_t J, uint32_t Rp, uint32_t* rec, uint32_t* ccount,
                      uint64_t nblk);
void launch_rec_fill(cudaStream_t s, const uint64_t* cpre, uint64_t nblk, uint32_t np, uint32_t J,
                     uint32_t Rp, uint32_t* rec, uint32_t nloc, uint32_t E, uint32_t MB,
                     uint32_t* cbase);
void launch_class_write(cudaStream_t s, const Part& part, uint32_t MB, const uint32_t* stream,
                        const uint32_t* rec, uint32_t np, uint32_t J, uint32_t Rp,
                        const uint32_t* cbase, const uint64_t* cstart, uint32_t* class_list,
                        uint64_t nblk);
void launch_class_lens(cudaStream_t s, uint32_t nloc, uint32_t E, uint32_t MB, uint32_t J,
                       const uint64_t* cpre, uint64_t nblk, uint64_t* clen);
void launch_holder_tile(cudaStream_t s, const Part& part, const uint32_t* inv, const uint16_t* rank16,
                        uint32_t MB, const uint32_t* rec, uint32_t np, uint32_t J, uint32_t Rp,
                        const uint32_t* cbase, const uint64_t* pair_off, uint32_t* holders,
                        bool allfit, const uint32_t* gate = nullptr);

}  // namespace clairplan
