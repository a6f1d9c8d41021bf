// Tier path of the dense seed build, laid out so that every random
// access of a pass hits a table that is L2-resident while the pass runs:
//
//   seg_write3   K4c  one CTA per (worker, epoch) segment, segments in epoch-major order (the
//                     CTAs in flight cover ~1 epoch, so the gathered info row of that epoch,
//                     28 MB at the ImageNet-22k shape, stays in L2).  Pass A: per-warp count
//                     histograms of the segment's first accesses (= its sub-range's offsets
//                     in the stable counting sort by count desc, policies.cpp:157-160); pass
//                     B (the segment re-read from L2): tier position of every candidate
//                     (dest), the sample id in tier order (sorted_k) and the block
//                     first-masks.  No size gather here (it used to stream the 114 MB sizes
//                     array through L2 next to everything else: 235 GB of DRAM reads).
//   gather_sizes      sorted_size[s] = sizes[sorted_k[s]]: the only traffic besides two
//                     streams is the size gather, so the sizes array stays L2-resident.
//   fill_class        a class whose capacity provably holds every remaining candidate of
//                     every worker (the whole-worker test of the all-fit path, against C_j):
//                     the first-fit chain of that class takes all of them, in any order.
//   hp_fill      K7b  hp[e][k] = class << 28 | class-list position of every first access,
//                     epoch-major: the block records of one epoch (7 MB at the ImageNet-22k
//                     shape) stay in L2 while that epoch's rows stream through.
//   holder_hp    K8   holder CSR sample-major from coalesced rows inv / rank / hp (no gather
//                     of block records over all epochs: 638 MB of random 16-B reads, 155 GB
//                     of DRAM traffic at the ImageNet-22k shape).
// Measured and dropped: hp written by the class-list pass (random u16/u32 writes into a
// 28-57 MB row per epoch: the partial sectors did not merge in L2, 43 GB of DRAM writes).
#include <algorithm>

#include "internal.h"

namespace clairplan {

constexpr uint32_t kSegWarps = 8;   // warps per segment CTA
constexpr int kSegU = 4;            // 32-entry blocks in flight per warp iteration

// ---------------------------------------------------------------------------- K4c
// STAGE >= 1: the segment's counts are kept in shared memory between the two passes (one info
// gather per entry); STAGE == 2: its sample ids too (the stream is read once, evict-first);
// STAGE == 0 (long segments): pass B reads the stream again and gathers the counts again.
constexpr uint32_t kStageMax = 49152;      // entries, counts staged

template <typename IT, int STAGE>
__global__ void __launch_bounds__(kSegWarps * 32) seg_write3_kernel(
    Part part, const uint32_t* __restrict__ stream, const IT* __restrict__ info,
    const uint64_t* __restrict__ seg_off, const uint64_t* __restrict__ sorted_base, uint32_t MB,
    uint32_t* __restrict__ dest, uint32_t* __restrict__ sorted_k, uint32_t* __restrict__ blkmask,
    uint32_t* __restrict__ blkbase, uint32_t* __restrict__ claim) {
    extern __shared__ uint32_t sm[];
    __shared__ uint32_t s_seg;  // [kSegWarps][E] count histograms -> offsets, [kSegWarps]
                                      // totals, STAGE: u8 count per segment entry
    const uint32_t E = part.E, nloc = part.wend - part.wbegin;
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t* hist = sm + warp * E;
    uint32_t* wtot = sm + kSegWarps * E;
    const uint64_t Lst = (uint64_t)MB * 32;  // staged entries per segment (max segment length)
    uint32_t* sk = sm + kSegWarps * E + kSegWarps;                          // STAGE 2: [Lst]
    IT* sc = reinterpret_cast<IT*>(sk + (STAGE == 2 ? Lst : 0));            // STAGE >= 1: [Lst]
    const uint64_t nseg = (uint64_t)nloc * E;
    // segments claimed in order from one counter (claim != null): the CTAs in flight stay within
    // ~one epoch however unevenly they progress (a fixed grid-stride assignment drifts apart
    // over the 90 epochs and the info rows of several epochs compete for L2)
    for (uint64_t seg = blockIdx.x;; seg += gridDim.x) {
        if (claim) {
            if (threadIdx.x == 0) s_seg = atomicAdd(claim, 1u);
            __syncthreads();
            seg = s_seg;
        }
        if (seg >= nseg) break;
        const uint32_t e = (uint32_t)(seg / nloc), wl = (uint32_t)(seg - (uint64_t)e * nloc);
        const uint32_t w = part.wbegin + wl;
        const uint64_t Le = part.epoch_len(w);
        const uint32_t nb = (uint32_t)((Le + 31) >> 5);
        const uint64_t g0 = part.stream_offset(w) + (uint64_t)e * Le;
        const IT* row = info + (size_t)e * part.Fp;
        const uint32_t b_lo = (uint32_t)(((uint64_t)nb * warp) / kSegWarps);
        const uint32_t b_hi = (uint32_t)(((uint64_t)nb * (warp + 1)) / kSegWarps);
        for (uint32_t i = lane; i < E; i += 32) hist[i] = 0;
        __syncwarp();
        // pass A: first accesses of the warp's blocks by count value (stream lines stay in L2)
        uint32_t tot = 0;
        for (uint32_t b0 = b_lo; b0 < b_hi; b0 += kSegU) {
            uint32_t k[kSegU], c[kSegU];
#pragma unroll
            for (int u = 0; u < kSegU; ++u) {
                const uint64_t t = (uint64_t)(b0 + u) * 32 + lane;
                if constexpr (STAGE == 2)
                    k[u] = (b0 + u < b_hi && t < Le) ? __ldcs(stream + g0 + t) : kNone;
                else
                    k[u] = (b0 + u < b_hi && t < Le) ? stream[g0 + t] : kNone;
            }
#pragma unroll
            for (int u = 0; u < kSegU; ++u) c[u] = k[u] == kNone ? 0u : (uint32_t)row[k[u]];
#pragma unroll
            for (int u = 0; u < kSegU; ++u) {
                if (STAGE >= 1 && b0 + u < b_hi) sc[(b0 + u) * 32 + lane] = (IT)c[u];
                if (STAGE == 2 && b0 + u < b_hi) sk[(b0 + u) * 32 + lane] = k[u];
                const bool first = c[u] != 0;
                const uint32_t key = first ? E - c[u] : (0x80000000u | lane);
                const uint32_t m = __match_any_sync(0xffffffffu, key);
                if (first && __popc(m & lanemask_lt()) == 0) hist[key] += __popc(m);
                tot += __popc(__ballot_sync(0xffffffffu, first));
            }
        }
        if (lane == 0) wtot[warp] = tot;
        __syncthreads();
        // exclusive scan down the warp axis, per count value: hist[w][i] = sum of warps < w
        for (uint32_t i = threadIdx.x; i < E; i += blockDim.x) {
            uint32_t run = 0;
#pragma unroll
            for (uint32_t q = 0; q < kSegWarps; ++q) {
                const uint32_t v = sm[q * E + i];
                sm[q * E + i] = run;
                run += v;
            }
        }
        uint32_t fpre = 0;
#pragma unroll
        for (uint32_t q = 0; q < kSegWarps; ++q) fpre += q < warp ? wtot[q] : 0u;
        __syncthreads();
        // pass B: tier positions, sample ids in tier order, block first-masks
        const uint64_t fbase = seg_off[(uint64_t)wl * E + e] + fpre;
        const uint64_t* sbase = sorted_base + (uint64_t)wl * E * E + e;  // + (E-c)*E
        const uint64_t blk0 = ((uint64_t)wl * E + e) * MB;
        uint64_t frun = 0;
        for (uint32_t b0 = b_lo; b0 < b_hi; b0 += kSegU) {
            uint32_t k[kSegU], c[kSegU];
#pragma unroll
            for (int u = 0; u < kSegU; ++u) {
                const uint64_t t = (uint64_t)(b0 + u) * 32 + lane;
                if constexpr (STAGE == 2)
                    k[u] = b0 + u < b_hi ? sk[(b0 + u) * 32 + lane] : kNone;
                else
                    k[u] = (b0 + u < b_hi && t < Le) ? __ldcs(stream + g0 + t) : kNone;  // last use
            }
#pragma unroll
            for (int u = 0; u < kSegU; ++u) {
                if constexpr (STAGE >= 1) c[u] = b0 + u < b_hi ? (uint32_t)sc[(b0 + u) * 32 + lane] : 0u;
                else c[u] = k[u] == kNone ? 0u : (uint32_t)row[k[u]];
                if (k[u] == kNone) c[u] = 0;
            }
#pragma unroll
            for (int u = 0; u < kSegU; ++u) {
                const uint32_t bi = b0 + u;
                if (bi >= b_hi) break;
                const bool first = c[u] != 0;
                const uint32_t bal = __ballot_sync(0xffffffffu, first);
                if (lane == 0) {
                    blkmask[blk0 + bi] = bal;
                    blkbase[blk0 + bi] = (uint32_t)(fbase + frun);
                }
                const uint32_t key = first ? E - c[u] : (0x80000000u | lane);
                const uint32_t m = __match_any_sync(0xffffffffu, key);
                const uint32_t leader = __ffs(m) - 1;
                uint32_t r0 = 0;
                if (first && lane == leader) {
                    r0 = hist[key];
                    hist[key] = r0 + __popc(m);
                }
                r0 = __shfl_sync(0xffffffffu, r0, leader);
                if (first) {
                    const uint64_t fpos = fbase + frun + __popc(bal & lanemask_lt());
                    const uint64_t spos = sbase[(uint64_t)key * E] + r0 + __popc(m & lanemask_lt());
                    __stcs(dest + fpos, (uint32_t)spos);
                    __stcs(sorted_k + spos, k[u]);
                }
                frun += __popc(bal);
            }
        }
        __syncthreads();  // hist / wtot / sc are reused by the next segment
    }
}

template <typename IT>
static void seg_write3_launch(cudaStream_t s, const Part& part, const uint32_t* stream, const IT* info,
                              const uint64_t* seg_off, const uint64_t* sorted_base, uint32_t MB,
                              uint32_t* dest, uint32_t* sorted_k, uint32_t* blkmask, uint32_t* blkbase,
                              uint32_t* claim) {
    const uint64_t nseg = (uint64_t)(part.wend - part.wbegin) * part.E;
    const uint64_t Lmax = (uint64_t)MB * 32;
    const size_t hbytes = (size_t)(kSegWarps * part.E + kSegWarps) * 4;
    // (staging the sample ids too, STAGE 2, measured slower at the ImageNet-22k shape: 72 KB of
    // shared memory per CTA left 3 CTAs per SM, 34 vs 13 ms)
    const int stage = Lmax <= kStageMax ? 1 : 0;
    const size_t smem = hbytes + (stage == 2 ? Lmax * (4 + sizeof(IT)) : stage == 1 ? Lmax * sizeof(IT) : 0);
    // every CTA resident, segments taken in epoch-major order: the CTAs in flight span under
    // one epoch of segments, so that epoch's info row stays in L2
#define SW3(ST)                                                                                   \
    do {                                                                                          \
        allow_smem(seg_write3_kernel<IT, ST>, \
                             (int)smem);                                                          \
        const unsigned grid = std::min<unsigned>(                                                 \
            resident_grid(seg_write3_kernel<IT, ST>, kSegWarps * 32, smem, 4), (unsigned)nseg);   \
        seg_write3_kernel<IT, ST><<<grid, kSegWarps * 32, smem, s>>>(                             \
            part, stream, info, seg_off, sorted_base, MB, dest, sorted_k, blkmask, blkbase, claim); \
    } while (0)
    if (stage == 1) SW3(1);
    else SW3(0);
#undef SW3
}

void launch_seg_write3(cudaStream_t s, const Part& part, const uint32_t* stream, const void* info,
                       bool info8, const uint64_t* seg_off, const uint64_t* sorted_base, uint32_t MB,
                       uint32_t* dest, uint32_t* sorted_k, uint32_t* blkmask, uint32_t* blkbase,
                       uint32_t* claim) {
    static const bool dyn = ab_knob("CLAIRPLAN_DYN", 1) != 0;  // A/B: fixed grid-stride order
    if (claim && dyn) cudaMemsetAsync(claim, 0, 4, s);
    if (!dyn) claim = nullptr;
    if (info8)
        seg_write3_launch(s, part, stream, static_cast<const uint8_t*>(info), seg_off, sorted_base, MB,
                          dest, sorted_k, blkmask, blkbase, claim);
    else
        seg_write3_launch(s, part, stream, static_cast<const uint16_t*>(info), seg_off, sorted_base, MB,
                          dest, sorted_k, blkmask, blkbase, claim);
}

// ---------------------------------------------------------------------------- sizes
__global__ void __launch_bounds__(kThreads) gather_sizes_kernel(const uint32_t* __restrict__ idx,
                                                                const double* __restrict__ sizes,
                                                                uint64_t n, double* __restrict__ out) {
    constexpr int U = 4;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x * U;
    for (uint64_t i0 = ((uint64_t)blockIdx.x * blockDim.x) * U + threadIdx.x; i0 < n; i0 += stride) {
        uint32_t k[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint64_t i = i0 + (uint64_t)u * blockDim.x;
            k[u] = i < n ? __ldcs(idx + i) : 0u;
        }
        double v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = __ldg(sizes + k[u]);
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint64_t i = i0 + (uint64_t)u * blockDim.x;
            if (i < n) __stcs(out + i, v[u]);
        }
    }
}

void launch_gather_sorted_sizes(cudaStream_t s, const uint32_t* sorted_k, const double* sizes,
                                uint64_t n, double* out) {
    gather_sizes_kernel<<<grid_for(n, kThreads * 4, 148u * 16u), kThreads, 0, s>>>(sorted_k, sizes, n, out);
}

// cls[s] = j where cls[s] == 0 (every remaining candidate fits class j)
__global__ void fill_class_kernel(uint8_t* __restrict__ cls, uint64_t n, uint8_t j) {
    const uint64_t n16 = n / 16;
    uint4* c4 = reinterpret_cast<uint4*>(cls);
    const uint32_t rep = 0x01010101u * j;
    for (uint64_t x = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; x < n16;
         x += (uint64_t)gridDim.x * blockDim.x) {
        uint4 v = c4[x];
        uint32_t* w = reinterpret_cast<uint32_t*>(&v);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            // per byte: zero -> j
            uint32_t z = w[q];
            uint32_t nz = ((z & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | z;  // high bit set where byte != 0
            nz = (nz >> 7) & 0x01010101u;                         // 1 where byte != 0
            const uint32_t zero_bytes = (0x01010101u - nz) * 0xFFu;  // 0xFF where byte == 0
            w[q] = z | (rep & zero_bytes);
        }
        c4[x] = v;
    }
    for (uint64_t x = n16 * 16 + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; x < n;
         x += (uint64_t)gridDim.x * blockDim.x)
        if (cls[x] == 0) cls[x] = j;
}

void launch_fill_class(cudaStream_t s, uint8_t* cls, uint64_t n, uint8_t j) {
    fill_class_kernel<<<grid_for(n / 16 + 1, kThreads, 148u * 16u), kThreads, 0, s>>>(cls, n, j);
}

// ---------------------------------------------------------------------------- K7b
// hp[e][k] = class << 28 | class-list position of the (e, k) first access (0: not a first
// access of this handle, or not cached).  Epoch-major, sample-major within the epoch: the
// block records gathered for epoch e (nloc * MB records, 7 MB at the ImageNet-22k shape) stay
// in L2 while the epoch's rows stream through; inv / rank rows are read and hp rows written
// coalesced.  The holder pass then needs no gather at all.
constexpr int kHpU = 8;  // consecutive samples per thread: 8 independent record gathers in flight

template <int NP>  // class bit-planes per record (0: runtime np)
__global__ void __launch_bounds__(kThreads, 3) hp_fill_kernel(Part part, const uint32_t* __restrict__ inv,
                                                           const uint16_t* __restrict__ rank16,
                                                           uint32_t MB, const uint32_t* __restrict__ rec,
                                                           uint32_t np, uint32_t J, uint32_t Rp,
                                                           const uint32_t* __restrict__ cbase,
                                                           uint32_t* __restrict__ hp,
                                                           uint32_t* __restrict__ claim) {
    const uint32_t E = part.E, F = part.F;
    const uint32_t nq = (F + kHpU - 1) / kHpU;  // groups of kHpU samples per row
    const uint64_t total = (uint64_t)E * nq;
    __shared__ uint32_t s_chunk;
    // chunks of blockDim groups claimed in order (claim != null): the CTAs stay within one
    // epoch's records; else a fixed grid-stride order
    for (uint64_t x0 = (uint64_t)blockIdx.x * blockDim.x;; x0 += (uint64_t)gridDim.x * blockDim.x) {
        if (claim) {
            __syncthreads();
            if (threadIdx.x == 0) s_chunk = atomicAdd(claim, 1u);
            __syncthreads();
            x0 = (uint64_t)s_chunk * blockDim.x;
        }
        if (x0 >= total) break;
        const uint64_t x = x0 + threadIdx.x;
        if (x >= total) continue;
        const uint32_t e = (uint32_t)(x / nq);
        const uint32_t k0 = (uint32_t)(x - (uint64_t)e * nq) * kHpU;
        // rank row: one 16-B load (rows pitched to Fp, a multiple of 16 samples)
        const uint4 rv = __ldcs(reinterpret_cast<const uint4*>(rank16 + (size_t)e * part.Fp + k0));
        const uint32_t rw[4] = {rv.x, rv.y, rv.z, rv.w};
        // inv row: two 16-B loads (same pitch; k0 + kHpU <= Fp)
        const uint4* iv4 = reinterpret_cast<const uint4*>(inv + (size_t)e * part.Fp + k0);
        const uint4 i0 = __ldcs(iv4), i1 = __ldcs(iv4 + 1);
        const uint32_t iw[kHpU] = {i0.x, i0.y, i0.z, i0.w, i1.x, i1.y, i1.z, i1.w};
        uint32_t p[kHpU];
#pragma unroll
        for (int u = 0; u < kHpU; ++u) {
            const uint32_t rk = (rw[u >> 1] >> ((u & 1) * 16)) & 0xFFFFu;
            p[u] = (k0 + u < F && rk != 0xFFFFu) ? iw[u] : kNone;
        }
        // per sample: its record (16 B) and (local worker << 5 | bit in the block) -- the
        // record row is recomputed in the rare case it is needed again (registers: no spills)
        uint4 a[kHpU];
        uint32_t wb[kHpU];
#pragma unroll
        for (int u = 0; u < kHpU; ++u) {
            if (p[u] == kNone) continue;
            uint32_t w;
            const uint32_t t = part.within_epoch(p[u], w);
            wb[u] = ((w - part.wbegin) << 5) | (t & 31);
            a[u] = __ldg(reinterpret_cast<const uint4*>(
                rec + rec_index(w - part.wbegin, e, part.wend - part.wbegin, MB, t >> 5) * Rp));
        }
        uint32_t out[kHpU];
#pragma unroll
        for (int u = 0; u < kHpU; ++u) {
            out[u] = 0;
            if (p[u] == kNone) continue;
            const uint32_t bit = wb[u] & 31, wl = wb[u] >> 5;
            const uint32_t npv = NP > 0 ? (uint32_t)NP : np;
            uint32_t cls = 0, cm = 0xffffffffu;
#pragma unroll
            for (uint32_t q = 0; q < (NP > 0 ? (uint32_t)NP : 4u); ++q) {
                if (q >= npv) break;
                const uint32_t pl = q == 0 ? a[u].x : q == 1 ? a[u].y : q == 2 ? a[u].z : a[u].w;
                cls |= ((pl >> bit) & 1u) << q;
            }
#pragma unroll
            for (uint32_t q = 0; q < (NP > 0 ? (uint32_t)NP : 4u); ++q) {
                if (q >= npv) break;
                const uint32_t pl = q == 0 ? a[u].x : q == 1 ? a[u].y : q == 2 ? a[u].z : a[u].w;
                cm &= ((cls >> q) & 1u) ? pl : ~pl;
            }
            if (cls) {
                const uint32_t wi = npv + cls - 1;
                uint32_t prew;
                if (wi < 4) {
                    prew = wi == 0 ? a[u].x : wi == 1 ? a[u].y : wi == 2 ? a[u].z : a[u].w;
                } else {
                    uint32_t w;
                    const uint32_t t = part.within_epoch(p[u], w);
                    prew = __ldg(rec + rec_index(wl, e, part.wend - part.wbegin, MB, t >> 5) * Rp + wi);
                }
                const uint32_t pos = prew - __ldg(cbase + wl * J + cls - 1) + __popc(cm & ((1u << bit) - 1u));
                out[u] = (cls << 28) | pos;
            }
        }
        uint4* dst = reinterpret_cast<uint4*>(hp + (size_t)e * part.Fp + k0);
        __stcs(dst, make_uint4(out[0], out[1], out[2], out[3]));
        __stcs(dst + 1, make_uint4(out[4], out[5], out[6], out[7]));
    }
}

void launch_hp_fill(cudaStream_t s, const Part& part, const uint32_t* inv, const uint16_t* rank16,
                    uint32_t MB, const uint32_t* rec, uint32_t np, uint32_t J, uint32_t Rp,
                    const uint32_t* cbase, uint32_t* hp, uint32_t* claim) {
    const uint64_t total = (uint64_t)part.E * ((part.F + kHpU - 1) / kHpU);
    // resident grid: epochs in lockstep, so one epoch's records stay in L2
    // (72 registers at 3 CTAs/SM: no spills; 2 CTAs/SM measured the same, 4 spills)
    static const bool dyn = ab_knob("CLAIRPLAN_DYN", 1) != 0;
    if (claim && dyn) cudaMemsetAsync(claim, 0, 4, s);
#define HPF(NPV)                                                                                   \
    do {                                                                                           \
        const unsigned grid = std::min<unsigned>(resident_grid(hp_fill_kernel<NPV>, kThreads, 0, 8), \
                                                 grid_for(total, kThreads, 148u * 64u));           \
        hp_fill_kernel<NPV><<<grid, kThreads, 0, s>>>(part, inv, rank16, MB, rec, np, J, Rp, cbase, hp, \
                                                      dyn ? claim : nullptr);                      \
    } while (0)
    if (np == 1) HPF(1);
    else if (np == 2) HPF(2);
    else HPF(0);
#undef HPF
}

// ---------------------------------------------------------------------------- K8
// CTA = 32 samples: inv / rank / hp rows of the tile into padded shared tiles (16-B / 8-B
// vector loads of the pitched rows; a TMA-box variant measured slower: DESIGN.md §4), then a warp per sample, lanes = epochs: every first access (rank != 0xFFFF)
// writes {worker, class, position} at pair_off[k] + rank (build_index order,
// policies.cpp:124-142).  Class 0 (not cached) records are compacted out afterwards if any.
template <int TU = 4>
__global__ void __launch_bounds__(kThreads) holder_hp_kernel(Part part, const uint32_t* __restrict__ inv,
                                                             const uint16_t* __restrict__ rank16,
                                                             const uint32_t* __restrict__ hp,
                                                             const uint64_t* __restrict__ pair_off,
                                                             uint32_t* __restrict__ holders) {
    extern __shared__ uint32_t sm[];
    const uint32_t E = part.E, F = part.F;
    uint32_t* tinv = sm;                                             // [E][33]
    uint32_t* thp = sm + (size_t)E * 33;                             // [E][33]
    uint16_t* trk = reinterpret_cast<uint16_t*>(sm + (size_t)2 * E * 33);  // [E][33]
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
    for (uint64_t k0 = (uint64_t)blockIdx.x * 32; k0 < F; k0 += (uint64_t)gridDim.x * 32) {
        __syncthreads();
        // thread per (epoch, quad of 4 samples): 16-B inv / hp loads and an 8-B rank load
        // (rows pitched to Fp: a quad that starts below F lies inside its row)
        for (uint32_t i0 = threadIdx.x; i0 < E * 8; i0 += TU * blockDim.x) {
            uint4 iv[TU], hv[TU];
            uint2 rv[TU];
#pragma unroll
            for (int u = 0; u < TU; ++u) {
                const uint32_t idx = i0 + u * blockDim.x;
                const uint32_t e = idx >> 3, l = (idx & 7) * 4;
                const bool ok = idx < E * 8 && k0 + l < F;
                const size_t o = (size_t)e * part.Fp + k0 + l;
                rv[u] = ok ? __ldcs(reinterpret_cast<const uint2*>(rank16 + o)) : make_uint2(~0u, ~0u);
                iv[u] = ok ? __ldcs(reinterpret_cast<const uint4*>(inv + o)) : make_uint4(kNone, kNone, kNone, kNone);
                hv[u] = ok ? __ldcs(reinterpret_cast<const uint4*>(hp + o)) : make_uint4(0, 0, 0, 0);
            }
#pragma unroll
            for (int u = 0; u < TU; ++u) {
                const uint32_t idx = i0 + u * blockDim.x;
                if (idx < E * 8) {
                    const uint32_t e = idx >> 3, l = (idx & 7) * 4;
                    uint32_t* ti = tinv + e * 33 + l;
                    uint32_t* th = thp + e * 33 + l;
                    uint16_t* tr = trk + e * 33 + l;
                    ti[0] = iv[u].x, ti[1] = iv[u].y, ti[2] = iv[u].z, ti[3] = iv[u].w;
                    th[0] = hv[u].x, th[1] = hv[u].y, th[2] = hv[u].z, th[3] = hv[u].w;
                    tr[0] = (uint16_t)rv[u].x, tr[1] = (uint16_t)(rv[u].x >> 16);
                    tr[2] = (uint16_t)rv[u].y, tr[3] = (uint16_t)(rv[u].y >> 16);
                }
            }
        }
        __syncthreads();
        for (uint32_t s = warp; s < 32; s += nwarps) {
            if (k0 + s >= F) break;
            const uint64_t slot0 = pair_off[k0 + s];
            for (uint32_t e = lane; e < E; e += 32) {
                const uint32_t rk = trk[e * 33 + s];
                if (rk == 0xFFFFu) continue;
                const uint32_t v = thp[e * 33 + s];
                uint32_t* h = holders + 3 * (slot0 + rk);
                __stcs(h, part.worker_of(tinv[e * 33 + s]));
                __stcs(h + 1, v >> 28);
                __stcs(h + 2, v & 0x0FFFFFFFu);
            }
        }
    }
}

bool holder_hp_ok(const Part& part) {  // the padded tiles fit one CTA's shared memory
    return (size_t)part.E * 33 * 4 * 2 + (size_t)part.E * 33 * 2 + 16 <= (200u << 10);
}

void launch_holder_hp(cudaStream_t s, const Part& part, const uint32_t* inv, const uint16_t* rank16,
                      const uint32_t* hp, const uint64_t* pair_off, uint32_t* holders) {
    const size_t smem = (size_t)part.E * 33 * 4 * 2 + (size_t)part.E * 33 * 2 + 16;
    const uint64_t tiles = ((uint64_t)part.F + 31) / 32;
    allow_smem(holder_hp_kernel<4>, (int)smem);
    holder_hp_kernel<4><<<grid_for(tiles, 1, 148u * 8u), kThreads, smem, s>>>(part, inv, rank16, hp,
                                                                              pair_off, holders);
}

}  // namespace clairplan
