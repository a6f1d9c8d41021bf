// Seed-path kernels of the plan build after the permutations (K4-K8), v2.
//
// Data layout (one handle = a worker range [wb, we), nloc workers):
//   inv   [E][F]  u32  position of sample k in epoch e's permutation (K3 output)
//   info  [E][Fp] u16  access count of (w,k) at the epoch of its first access, else 0
//   rank  [E][Fp] u16  rank of w among k's workers at that access, else 0xFFFF
//                      (Fp = F rounded up to 8: 16-B aligned rows)
//   stream         u32 worker-major access streams; segment (w,e) = worker w's epoch e,
//                      contiguous, length Le(w); split into 32-entry blocks
//                      blk(w,e,t) = ((w-wb)*E + e)*MB + t/32, MB = ceil(max Le / 32)
//   candidates     per worker in first-access order ("first order", c)   -- dest[c]
//   sorted         per worker in tier order (count desc, first asc)      -- sorted_size[s]
//   block records  blkmask/blkbase (first-access bits, first-order index of the first one),
//                  np class bit-planes and per-class prefix counts; all-fit path: uint2
//                  {first-access mask, worker-local first-order index}
//
// K4a sample_tile    CTA = 32 samples, warp per sample, lanes = epochs; per-warp shared
//                    tables (first epoch, count, worker bitmap) -> info / rank, pair counts,
//                    per-worker candidate size sums (all-fit test).  sample_lanes /
//                    sample_hash: fallbacks for nloc > 1024 or E > 128.
// all-fit seg_allfit one pass: class-1 lists + block records, decoupled look-back (§4.3)
// K4b seg_hist       per (w,e) segment: histogram of first accesses by count (tier path)
// K4c seg_write      per segment: first-order index, tier-order index (stable counting sort
//                    by count desc = policies.cpp:157-160), sizes gathered in tier order,
//                    block first-masks
// K7  blk_codes      class bit-planes + per-class counts per block (after first fit)
//     class_write    prefetch-ordered class lists (policies.cpp:31-36,162)
// K8  holder_tile    CTA = 32 samples, warp per sample: holders written in worker order at
//                    the pair slot (build_index, policies.cpp:124-142) from the block records
#include <math.h>
#include <stdlib.h>

#include <type_traits>

#include "internal.h"

namespace clairplan {

constexpr int kU = 8;         // epochs loaded per batch (memory-level parallelism)

__device__ __forceinline__ uint32_t ld_inv(const uint32_t* p) { return __ldcs(p); }

// ---------------------------------------------------------------------------- K4a
// Lane = sample, everything per lane in shared memory with a [row][lane] layout (no bank
// conflicts).  Pass 1 streams the E inverse entries (kU coalesced loads in flight) and records
// the worker of every access (bit 15 = first access of that worker) while marking a per-lane
// worker bitmap; after its popcount prefix, pass 2 counts accesses per rank, pass 3 writes
//   info[e][k] = count of (w,k) at its first epoch, else 0          (u16)
//   rank[e][k] = rank of w among k's workers (worker order), else 0xFFFF  (u16)
__global__ void __launch_bounds__(128) sample_lanes_kernel(Part part, const uint32_t* __restrict__ inv,
                                                           uint16_t* __restrict__ info,
                                                           uint16_t* __restrict__ rank16,
                                                           uint32_t* __restrict__ pair_count,
                                                           uint32_t W,
                                                           uint32_t* __restrict__ seghist) {
    extern __shared__ uint32_t sm[];
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t E = part.E, F = part.F;
    const uint32_t per_warp = 64 * W + 32 * E;  // words: bm, pre, wls (u16), cnt (u16)
    uint32_t* bm = sm + warp * per_warp;  // [W][32]
    uint32_t* pre = bm + 32 * W;          // [W][32]
    uint16_t* wls = reinterpret_cast<uint16_t*>(pre + 32 * W);  // [E][32]
    uint16_t* cnt = wls + 32 * E;                                // [E][32] by rank
    for (uint32_t t = 0; t < W; ++t) bm[t * 32 + lane] = 0;
    const uint64_t ngroups = (F + 31) / 32;
    const uint64_t gw = (uint64_t)blockIdx.x * (blockDim.x >> 5) + warp;
    const uint64_t nw = (uint64_t)gridDim.x * (blockDim.x >> 5);
    for (uint64_t g = gw; g < ngroups; g += nw) {
        const uint32_t k = (uint32_t)(g * 32 + lane);
        const bool live = k < F;
        for (uint32_t e0 = 0; e0 < E; e0 += kU) {
            uint32_t pv[kU];
#pragma unroll
            for (int u = 0; u < kU; ++u)
                pv[u] = (live && e0 + u < E) ? ld_inv(inv + (size_t)(e0 + u) * part.Fp + k) : kNone;
#pragma unroll
            for (int u = 0; u < kU; ++u) {
                const uint32_t e = e0 + u;
                if (e >= E) break;
                uint32_t rec = 0xFFFFu;
                const uint32_t p = pv[u];
                if (p < part.P) {
                    const uint32_t w = part.worker_of(p);
                    if (w >= part.wbegin && w < part.wend) {
                        const uint32_t wl = w - part.wbegin;
                        uint32_t* word = &bm[(wl >> 5) * 32 + lane];
                        const uint32_t bit = 1u << (wl & 31);
                        const uint32_t v = *word;
                        *word = v | bit;
                        rec = wl | ((v & bit) ? 0u : 0x8000u);
                    }
                }
                wls[e * 32 + lane] = (uint16_t)rec;
            }
        }
        uint32_t d = 0;
        for (uint32_t t = 0; t < W; ++t) {
            pre[t * 32 + lane] = d;
            d += __popc(bm[t * 32 + lane]);
        }
        if (live) pair_count[k] = d;
        for (uint32_t r = 0; r < d; ++r) cnt[r * 32 + lane] = 0;
        for (uint32_t e = 0; e < E; ++e) {
            const uint32_t rec = wls[e * 32 + lane];
            if (rec == 0xFFFFu) continue;
            const uint32_t wl = rec & 0x7FFFu, wd = (wl >> 5) * 32 + lane;
            const uint32_t r = pre[wd] + __popc(bm[wd] & ((1u << (wl & 31)) - 1u));
            cnt[r * 32 + lane] += 1;
        }
        if (live) {
            for (uint32_t e = 0; e < E; ++e) {
                const uint32_t rec = wls[e * 32 + lane];
                uint16_t c = 0, rk = 0xFFFFu;
                if (rec != 0xFFFFu && (rec & 0x8000u)) {
                    const uint32_t wl = rec & 0x7FFFu, wd = (wl >> 5) * 32 + lane;
                    const uint32_t r = pre[wd] + __popc(bm[wd] & ((1u << (wl & 31)) - 1u));
                    c = cnt[r * 32 + lane];
                    rk = (uint16_t)r;
                    // per-(worker, epoch) segment histogram of first accesses by count
                    if (seghist) atomicAdd(&seghist[((uint64_t)wl * E + (E - c)) * E + e], 1u);
                }
                __stcs(info + (size_t)e * part.Fp + k, c);
                __stcs(rank16 + (size_t)e * part.Fp + k, rk);
            }
        }
        for (uint32_t t = 0; t < W; ++t) bm[t * 32 + lane] = 0;
    }
}

// Exact fallback for samples whose repeated-worker list overflowed (and for handles with
// more than kMaxLaneWorkers workers): one warp per sample, __match_any_sync per 32-epoch
// round + a per-warp shared-memory hash keyed by worker.
__global__ void __launch_bounds__(128) sample_hash_kernel(Part part, const uint32_t* __restrict__ inv,
                                                          uint16_t* __restrict__ info,
                                                          uint16_t* __restrict__ rank16,
                                                          uint32_t* __restrict__ pair_count,
                                                          const uint32_t* __restrict__ list,
                                                          const uint32_t* __restrict__ nlist,
                                                          uint32_t hs, uint32_t W,
                                                          uint32_t* __restrict__ seghist) {
    extern __shared__ uint32_t sm[];
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t* keys = sm + warp * (2 * hs + 2 * W);
    uint32_t* vals = keys + hs;
    uint32_t* bm = vals + hs;   // [W] workers of the current sample
    uint32_t* pre = bm + W;     // [W] popcount prefix
    const uint32_t mask = hs - 1;
    const uint32_t E = part.E, F = part.F;
    const uint32_t n = list ? *nlist : F;
    for (uint32_t t = lane; t < hs; t += 32) keys[t] = kNone;
    for (uint32_t t = lane; t < W; t += 32) bm[t] = 0;
    __syncwarp();
    for (uint32_t idx = blockIdx.x * (blockDim.x >> 5) + warp; idx < n;
         idx += gridDim.x * (blockDim.x >> 5)) {
        const uint32_t k = list ? list[idx] : idx;
        uint32_t distinct = 0;
        for (uint32_t r = 0; r * 32 < E; ++r) {
            const uint32_t e = r * 32 + lane;
            uint32_t w = kNone;
            if (e < E) {
                const uint32_t p = inv[(size_t)e * part.Fp + k];
                if (p < part.P) {
                    const uint32_t ww = part.worker_of(p);
                    if (ww >= part.wbegin && ww < part.wend) w = ww - part.wbegin;
                }
            }
            const uint32_t m = __match_any_sync(0xffffffffu, w);
            const bool leader = (__ffs(m) - 1) == (int)lane;
            bool fresh = false;
            if (w != kNone && leader) {
                uint32_t slot = (w * 0x9E3779B1u >> 7) & mask;
                while (true) {
                    const uint32_t old = atomicCAS(&keys[slot], kNone, w);
                    if (old == kNone) {
                        vals[slot] = (e << 16) | __popc(m);
                        fresh = true;
                        break;
                    }
                    if (old == w) {
                        vals[slot] += __popc(m);
                        break;
                    }
                    slot = (slot + 1) & mask;
                }
                if (fresh) atomicOr(&bm[w >> 5], 1u << (w & 31));
            }
            distinct += __popc(__ballot_sync(0xffffffffu, fresh));
            __syncwarp();
        }
        {   // prefix popcounts of the worker bitmap (lane-strided words, warp scan)
            uint32_t carry = 0;
            for (uint32_t t0 = 0; t0 < W; t0 += 32) {
                const uint32_t t = t0 + lane;
                const uint32_t c = t < W ? __popc(bm[t]) : 0;
                uint32_t incl = c;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
                    if ((int)lane >= o) incl += y;
                }
                if (t < W) pre[t] = carry + incl - c;
                carry += __shfl_sync(0xffffffffu, incl, 31);
            }
        }
        __syncwarp();
        for (uint32_t r = 0; r * 32 < E; ++r) {
            const uint32_t e = r * 32 + lane;
            if (e >= E) continue;
            const uint32_t p = inv[(size_t)e * part.Fp + k];
            uint16_t out = 0, rk = 0xFFFFu;
            if (p < part.P) {
                const uint32_t ww = part.worker_of(p);
                if (ww >= part.wbegin && ww < part.wend) {
                    const uint32_t w = ww - part.wbegin;
                    uint32_t slot = (w * 0x9E3779B1u >> 7) & mask;
                    while (keys[slot] != w) slot = (slot + 1) & mask;
                    const uint32_t v = vals[slot];
                    if ((v >> 16) == e) {
                        out = (uint16_t)(v & 0xFFFFu);
                        rk = (uint16_t)(pre[w >> 5] + __popc(bm[w >> 5] & ((1u << (w & 31)) - 1u)));
                        if (seghist) atomicAdd(&seghist[((uint64_t)w * E + (E - out)) * E + e], 1u);
                    }
                }
            }
            info[(size_t)e * part.Fp + k] = out;
            rank16[(size_t)e * part.Fp + k] = rk;
        }
        __syncwarp();
        for (uint32_t t = lane; t < hs; t += 32) keys[t] = kNone;
        for (uint32_t t = lane; t < W; t += 32) bm[t] = 0;
        if (lane == 0) pair_count[k] = distinct;
        __syncwarp();
    }
}

// ---------------------------------------------------------------------------- K4b
// One warp per (worker, epoch) segment; kSU 32-entry steps are loaded ahead (stream words,
// then their info words — the join with the sample pass, L2-resident per epoch because the
// segments are ordered epoch-major).  No block barriers: per-count counters live in the
// warp's shared slice, one leader per count value per step (__match_any_sync).
constexpr int kSU = 4;

// seghist[(wl*E + (E - c))*E + e] = first accesses with count c in segment (w, e)
// With `sizes`: also the sum and minimum of the sizes of the segment's first accesses
// (segsum/segmin), the input of the whole-worker fit test (fit_check_kernel).
// seghist[(wl*E + (E - c))*E + e] = first accesses with count c in segment (w, e)
template <typename IT>
__global__ void __launch_bounds__(kThreads) seg_hist_kernel(Part part, const uint32_t* __restrict__ stream,
                                                             const IT* __restrict__ info,
                                                             const uint32_t* __restrict__ cpos,
                                                             uint32_t* __restrict__ seghist,
                                                             uint32_t* __restrict__ segcnt) {
    extern __shared__ uint32_t shist[];  // [warps][E]
    const uint32_t E = part.E, nloc = part.wend - part.wbegin;
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t* hist = shist + warp * E;
    const uint64_t nseg = (uint64_t)nloc * E;
    for (uint64_t b = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; b < nseg;
         b += ((uint64_t)gridDim.x * blockDim.x) >> 5) {
        const uint32_t e = (uint32_t)(b / nloc), wl = (uint32_t)(b - (uint64_t)e * nloc);
        const uint32_t w = part.wbegin + wl;
        for (uint32_t i = lane; i < E; i += 32) hist[i] = 0;
        __syncwarp();
        const uint64_t Le = part.epoch_len(w);
        const uint64_t g0 = part.stream_offset(w) + (uint64_t)e * Le;
        const IT* row = info + (size_t)e * part.Fp;
        uint32_t tot = 0;
        for (uint64_t t0 = 0; t0 < Le; t0 += 32 * kSU) {
            uint32_t k[kSU], c[kSU];
#pragma unroll
            for (int u = 0; u < kSU; ++u) {
                const uint64_t t = t0 + 32 * u + lane;
                k[u] = t < Le ? __ldcs(stream + g0 + t) : kNone;
            }
#pragma unroll
            for (int u = 0; u < kSU; ++u)
                c[u] = k[u] == kNone ? 0u : cpos ? info[cpos[g0 + t0 + 32 * u + lane]] : row[k[u]];
#pragma unroll
            for (int u = 0; u < kSU; ++u) {
                const bool first = c[u] != 0;
                const uint32_t key = first ? E - c[u] : (0x80000000u | lane);
                const uint32_t m = __match_any_sync(0xffffffffu, key);
                if (first && __popc(m & lanemask_lt()) == 0) hist[key] += __popc(m);
                tot += first;
            }
            __syncwarp();
        }
        tot = warp_sum(tot);
        __syncwarp();
        for (uint32_t i = lane; i < E; i += 32) seghist[((uint64_t)wl * E + i) * E + e] = hist[i];
        if (lane == 0) segcnt[(uint64_t)wl * E + e] = tot;
        __syncwarp();
    }
}

// per-segment first-access totals from the segment histograms (sum over count values)
__global__ void segcnt_kernel(uint32_t nloc, uint32_t E, const uint32_t* __restrict__ seghist,
                              uint32_t* __restrict__ segcnt) {
    for (uint64_t x = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; x < (uint64_t)nloc * E;
         x += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t wl = x / E, e = x % E;
        uint32_t s = 0;
        for (uint32_t i = 0; i < E; ++i) s += seghist[(wl * E + i) * E + e];
        segcnt[x] = s;
    }
}

void launch_segcnt(cudaStream_t s, uint32_t nloc, uint32_t E, const uint32_t* seghist,
                   uint32_t* segcnt) {
    segcnt_kernel<<<grid_for((uint64_t)nloc * E, kThreads), kThreads, 0, s>>>(nloc, E, seghist,
                                                                              segcnt);
}

// ---------------------------------------------------------------------------- all-fit path
// pack_first_fit (policies.cpp:40-55) takes every candidate of a worker into class 1 when the
// sizes are non-negative and their sum stays below the capacity by more than the rounding of
// any summation order and of the chain `remaining -= s`: `s <= remaining` then holds at every
// step whatever the tier order is.  The per-worker sums come from the sample pass
// (WorkerSums); the host decides (allfit_decide, plan.cu).  Then one pass over the streams:
//
// seg_allfit   warp per chunk of kAllfitChunk stream entries, chunks taken from a ticket
//              counter in epoch-major order (the info row of one epoch stays L2-resident).
//              Pass A: first accesses (ballots kept one per lane); the chunk's count is
//              published and the worker-local first-order prefix found by a decoupled
//              look-back over the worker's earlier chunks (all hold smaller tickets, so they
//              are running or done: no deadlock).  Pass B re-reads the chunk (L2) and writes
//              per 32-entry block the record {first-access mask, worker-local first-order
//              index} and the class-1 list (= first-access order = prefetch order) at the
//              worker's stream offset.
constexpr unsigned long long kStAgg = 1ull << 62, kStInc = 2ull << 62, kStMask = (1ull << 62) - 1;

template <typename IT>
__global__ void __launch_bounds__(kThreads) seg_allfit_kernel(
    Part part, const uint32_t* __restrict__ stream, const IT* __restrict__ info,
    const uint32_t* __restrict__ cpos, uint32_t MB, uint32_t C,
    unsigned long long* __restrict__ status, uint32_t* __restrict__ ticket,
    uint32_t* __restrict__ rec, uint32_t* __restrict__ class_list, const uint32_t* __restrict__ gate) {
    if (gate && *gate == 0) return;  // speculative launch, the all-fit test failed
    const uint32_t E = part.E, nloc = part.wend - part.wbegin;
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t nch = (uint64_t)nloc * E * C;
    while (true) {
        uint32_t tk = 0;
        if (lane == 0) tk = atomicAdd(ticket, 1u);
        tk = __shfl_sync(0xffffffffu, tk, 0);
        if (tk >= nch) break;
        const uint32_t e = (uint32_t)(tk / ((uint64_t)nloc * C));
        const uint32_t r = (uint32_t)(tk - (uint64_t)e * nloc * C);
        const uint32_t wl = r / C, ci = r - wl * C;
        const uint32_t w = part.wbegin + wl;
        const uint64_t Le = part.epoch_len(w);
        const uint64_t t_lo = (uint64_t)ci * kAllfitChunk;
        const uint64_t t_hi = t_lo + kAllfitChunk < Le ? t_lo + kAllfitChunk : Le;
        const uint64_t sw = part.stream_offset(w);
        const uint64_t g0 = sw + (uint64_t)e * Le;
        const IT* row = info + (size_t)e * part.Fp;
        const uint64_t x = ((uint64_t)wl * E + e) * C + ci;  // worker-major chunk index
        // pass A: first-access ballots, lane b keeps block b's
        uint32_t mymask = 0, tot = 0;
        for (uint64_t t0 = t_lo; t0 < t_hi; t0 += 32 * kSU) {
            uint32_t k[kSU], c[kSU];
#pragma unroll
            for (int u = 0; u < kSU; ++u) {
                const uint64_t t = t0 + 32 * u + lane;
                // kept in L2 for pass B (an evict-first load here made pass B re-read the
                // chunk from DRAM: +0.42 GB per config-2 plan)
                k[u] = t < t_hi ? stream[g0 + t] : kNone;
            }
#pragma unroll
            for (int u = 0; u < kSU; ++u)
                c[u] = k[u] == kNone ? 0u : cpos ? info[cpos[g0 + t0 + 32 * u + lane]] : row[k[u]];
#pragma unroll
            for (int u = 0; u < kSU; ++u) {
                const uint64_t tb = t0 + 32 * u;
                const uint32_t bal = __ballot_sync(0xffffffffu, c[u] != 0);
                if (tb < t_hi && lane == (uint32_t)((tb - t_lo) >> 5)) mymask = bal;
                tot += __popc(bal);
            }
        }
        // publish, then a warp-wide look-back over the worker's chain of chunks: lane j reads
        // chunk x-1-j, the window stops at the nearest inclusive prefix (the worker's first
        // chunk is always inclusive)
        unsigned long long prefix = 0;
        const uint64_t first_x = (uint64_t)wl * E * C;
        if (lane == 0) atomicExch(status + x, (x == first_x ? kStInc : kStAgg) | tot);
        if (x != first_x) {
            for (uint64_t j0 = x - 1;; j0 -= 32) {
                const bool valid = j0 >= first_x + lane;  // j0 - lane >= first_x
                unsigned long long v = 0;
                if (valid) {
                    do {
                        v = *reinterpret_cast<volatile unsigned long long*>(status + (j0 - lane));
                    } while (v == 0);
                }
                const uint32_t incm = __ballot_sync(0xffffffffu, valid && (v & kStInc));
                const uint32_t upto = incm ? (uint32_t)(__ffs(incm) - 1) : 31u;
                unsigned long long add = (valid && lane <= upto) ? (v & kStMask) : 0ull;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) add += __shfl_xor_sync(0xffffffffu, add, o);
                prefix += add;
                if (incm) break;
            }
            if (lane == 0) atomicExch(status + x, kStInc | (prefix + tot));
        }
        prefix = __shfl_sync(0xffffffffu, prefix, 0);
        // pass B: block records and the class-1 list
        uint64_t run = prefix;
        const uint64_t blk0 = rec_index(wl, e, nloc, MB, 0);
        for (uint64_t t0 = t_lo; t0 < t_hi; t0 += 32 * kSU) {
            uint32_t k[kSU];
#pragma unroll
            for (int u = 0; u < kSU; ++u) {
                const uint64_t t = t0 + 32 * u + lane;
                k[u] = t < t_hi ? __ldcs(stream + g0 + t) : kNone;  // last use
            }
#pragma unroll
            for (int u = 0; u < kSU; ++u) {
                const uint64_t tb = t0 + 32 * u;
                const uint32_t bal = __shfl_sync(0xffffffffu, mymask, (uint32_t)((tb - t_lo) >> 5) & 31);
                if (tb < t_hi) {
                    if (lane == 0)
                        reinterpret_cast<uint2*>(rec)[blk0 + (tb >> 5)] = make_uint2(bal, (uint32_t)run);
                    if ((bal >> lane) & 1u)
                        __stcs(class_list + sw + run + __popc(bal & lanemask_lt()), k[u]);
                    run += __popc(bal);
                }
            }
        }
    }
}

// class-list geometry of an all-fit handle: list (w, 1) = the worker's candidates at its stream
// offset, lists (w, j > 1) empty; class bases 0 (records hold worker-local indices)
__global__ void allfit_meta_kernel(Part part, uint32_t J, const uint32_t* __restrict__ wcnt,
                                   uint64_t* __restrict__ clen, uint64_t* __restrict__ cstart,
                                   uint32_t* __restrict__ cbase, const uint32_t* __restrict__ gate) {
    if (gate && *gate == 0) return;
    const uint32_t nloc = part.wend - part.wbegin;
    for (uint32_t x = blockIdx.x * blockDim.x + threadIdx.x; x <= nloc * J; x += gridDim.x * blockDim.x) {
        if (x == nloc * J) {
            cstart[x] = part.stream_offset(part.wend);
            break;
        }
        const uint32_t wl = x / J, j = x % J;
        const uint64_t a = part.stream_offset(part.wbegin + wl);
        clen[x] = j == 0 ? wcnt[wl] : 0;
        cstart[x] = j == 0 ? a : a + wcnt[wl];
        cbase[x] = 0;
    }
}

void launch_seg_allfit(cudaStream_t s, const Part& part, const uint32_t* stream, const void* info,
                       bool info8, const uint32_t* cpos, uint32_t MB, uint32_t C,
                       unsigned long long* status, uint32_t* ticket, uint32_t* rec,
                       uint32_t* class_list, const uint32_t* gate) {
    const uint64_t nch = (uint64_t)(part.wend - part.wbegin) * part.E * C;
    cudaMemsetAsync(status, 0, nch * 8, s);
    cudaMemsetAsync(ticket, 0, 4, s);
    const unsigned grid = grid_for(nch * 32, kThreads, 148u * 8u);
    if (info8)
        seg_allfit_kernel<uint8_t><<<grid, kThreads, 0, s>>>(
            part, stream, static_cast<const uint8_t*>(info), cpos, MB, C, status, ticket, rec, class_list, gate);
    else
        seg_allfit_kernel<uint16_t><<<grid, kThreads, 0, s>>>(
            part, stream, static_cast<const uint16_t*>(info), cpos, MB, C, status, ticket, rec, class_list, gate);
}

void launch_allfit_meta(cudaStream_t s, const Part& part, uint32_t J, const uint32_t* wcnt,
                        uint64_t* clen, uint64_t* cstart, uint32_t* cbase, const uint32_t* gate) {
    allfit_meta_kernel<<<grid_for((uint64_t)(part.wend - part.wbegin) * J + 1, kThreads), kThreads, 0, s>>>(
        part, J, wcnt, clen, cstart, cbase, gate);
}

// the whole-worker fit test of allfit_decide (plan.cu) on the device: *ok stays nonzero only
// when no size was negative and every worker's candidates fit class 1
__global__ void allfit_decide_kernel(uint32_t nloc, const unsigned long long* __restrict__ wsum,
                                     const uint32_t* __restrict__ wcnt, double C, uint32_t* ok) {
    for (uint32_t w = blockIdx.x * blockDim.x + threadIdx.x; w <= nloc; w += gridDim.x * blockDim.x) {
        if (w == nloc) {
            if (wcnt[nloc]) atomicAnd(ok, 0u);  // the negative-size flag
            continue;
        }
        if (wcnt[w] == 0) continue;
        const double sw = (double)wsum[w] * 0x1.0p-20;
        const double tol = ((double)wcnt[w] + 1024.0) * fmax(C, sw) * 0x1.0p-48;
        if (!(C - sw > tol)) atomicAnd(ok, 0u);
    }
}

void launch_allfit_decide(cudaStream_t s, uint32_t nloc, const unsigned long long* wsum,
                          const uint32_t* wcnt, double C, uint32_t* ok) {
    cudaMemsetAsync(ok, 0xFF, 4, s);
    allfit_decide_kernel<<<grid_for((uint64_t)nloc + 1, kThreads), kThreads, 0, s>>>(nloc, wsum, wcnt, C, ok);
}

// ---------------------------------------------------------------------------- K4c
template <typename IT>
__global__ void __launch_bounds__(kThreads) seg_write_kernel2(
    Part part, const uint32_t* __restrict__ stream, const IT* __restrict__ info, const uint32_t* __restrict__ cpos,
    const double* __restrict__ sizes, const uint64_t* __restrict__ seg_off,
    const uint64_t* __restrict__ sorted_base, uint32_t MB, uint32_t* __restrict__ dest,
    double* __restrict__ sorted_size, uint32_t* __restrict__ blkmask,
    uint32_t* __restrict__ blkbase) {
    extern __shared__ uint32_t srun[];  // [warps][E] running count per count value
    const uint32_t E = part.E, nloc = part.wend - part.wbegin;
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t* run = srun + warp * E;
    const uint64_t nseg = (uint64_t)nloc * E;
    for (uint64_t b = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; b < nseg;
         b += ((uint64_t)gridDim.x * blockDim.x) >> 5) {
        const uint32_t e = (uint32_t)(b / nloc), wl = (uint32_t)(b - (uint64_t)e * nloc);
        const uint32_t w = part.wbegin + wl;
        for (uint32_t i = lane; i < E; i += 32) run[i] = 0;
        __syncwarp();
        const uint64_t Le = part.epoch_len(w);
        const uint64_t g0 = part.stream_offset(w) + (uint64_t)e * Le;
        const IT* row = info + (size_t)e * part.Fp;
        const uint64_t fbase = seg_off[(uint64_t)wl * E + e];
        const uint64_t* sbase = sorted_base + (uint64_t)wl * E * E + e;  // + (E-c)*E
        const uint64_t blk0 = ((uint64_t)wl * E + e) * MB;
        uint64_t frun = 0;
        for (uint64_t t0 = 0; t0 < Le; t0 += 32 * kSU) {
            uint32_t k[kSU], c[kSU];
#pragma unroll
            for (int u = 0; u < kSU; ++u) {
                const uint64_t t = t0 + 32 * u + lane;
                k[u] = t < Le ? __ldcs(stream + g0 + t) : kNone;
            }
#pragma unroll
            for (int u = 0; u < kSU; ++u)
                c[u] = k[u] == kNone ? 0u : cpos ? info[cpos[g0 + t0 + 32 * u + lane]] : row[k[u]];
#pragma unroll
            for (int u = 0; u < kSU; ++u) {
                const uint64_t tb = t0 + 32 * u;
                if (tb >= Le) break;
                const bool first = c[u] != 0;
                const uint32_t bal = __ballot_sync(0xffffffffu, first);
                if (lane == 0) {
                    blkmask[blk0 + (tb >> 5)] = bal;
                    blkbase[blk0 + (tb >> 5)] = (uint32_t)(fbase + frun);
                }
                const uint32_t key = first ? E - c[u] : (0x80000000u | lane);
                const uint32_t m = __match_any_sync(0xffffffffu, key);
                const uint32_t leader = __ffs(m) - 1;
                uint32_t r0 = 0;
                if (first && lane == leader) {
                    r0 = run[key];
                    run[key] = r0 + __popc(m);
                }
                r0 = __shfl_sync(0xffffffffu, r0, leader);
                if (first) {
                    const uint64_t fpos = fbase + frun + __popc(bal & lanemask_lt());
                    const uint64_t spos = sbase[(uint64_t)key * E] + r0 + __popc(m & lanemask_lt());
                    __stcs(dest + fpos, (uint32_t)spos);
                    __stcs(sorted_size + spos, sizes[k[u]]);
                }
                frun += __popc(bal);
            }
            __syncwarp();
        }
        __syncwarp();
    }
}

// ---------------------------------------------------------------------------- K7
// Block record rec[blk][Rp], Rp = R rounded up to 4 words, R = np + J: np class bit-planes
// (bit p of the class of every first access of the block; class 0 = not cached / not a first
// access) followed by the J per-class prefix counts (class-j first accesses in all earlier
// blocks of the handle).  Four blocks per warp iteration keep the dependent gathers
// (mask -> first-order index -> tier position -> class) overlapped.
constexpr int kBU = 4;

// One warp per (worker, epoch) segment, kBU blocks per iteration: no per-block division and
// the dependent gathers (mask -> first-order index -> tier position -> class) of kBU blocks
// overlap.
template <int NJ>  // classes (0: runtime J); the bit-plane count follows
__global__ void __launch_bounds__(kThreads) blk_codes_kernel(
    Part part, uint32_t MB, const uint32_t* __restrict__ blkmask,
    const uint32_t* __restrict__ blkbase, const uint32_t* __restrict__ dest,
    const uint8_t* __restrict__ cls_sorted, uint32_t np_rt, uint32_t J_rt, uint32_t Rp,
    uint32_t* __restrict__ rec, uint32_t* __restrict__ ccount, uint64_t nblk) {
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t J = NJ > 0 ? (uint32_t)NJ : J_rt;
    const uint32_t np = NJ > 0 ? (NJ >= 4 ? 3u : NJ >= 2 ? 2u : 1u) : np_rt;
    const uint32_t E = part.E, nloc = part.wend - part.wbegin;
    const uint64_t nseg = (uint64_t)nloc * E;
    for (uint64_t seg = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; seg < nseg;
         seg += ((uint64_t)gridDim.x * blockDim.x) >> 5) {
        const uint32_t wl = (uint32_t)(seg / E);
        const uint32_t nb = (uint32_t)((part.epoch_len(part.wbegin + wl) + 31) >> 5);
        const uint64_t blk0 = seg * MB;
        const uint64_t rec0 = rec_index(wl, (uint32_t)(seg - (uint64_t)wl * E), nloc, MB, 0);
        for (uint32_t b0 = 0; b0 < MB; b0 += kBU) {
            uint32_t m[kBU], c[kBU], d[kBU], cls[kBU];
#pragma unroll
            for (int u = 0; u < kBU; ++u) {
                const uint32_t bi = b0 + u;
                m[u] = 0;
                if (bi < nb) {
                    m[u] = blkmask[blk0 + bi];
                    c[u] = blkbase[blk0 + bi];
                }
            }
#pragma unroll
            for (int u = 0; u < kBU; ++u)
                d[u] = ((m[u] >> lane) & 1u) ? dest[c[u] + __popc(m[u] & lanemask_lt())] : kNone;
#pragma unroll
            for (int u = 0; u < kBU; ++u) cls[u] = d[u] != kNone ? cls_sorted[d[u]] : 0u;
#pragma unroll
            for (int u = 0; u < kBU; ++u) {
                const uint32_t bi = b0 + u;
                if (bi >= MB) break;
                const uint64_t blk = blk0 + bi;
                uint32_t word = 0;  // lane p < np holds plane p, lane np + j holds count of class j+1
                if constexpr (NJ > 0) {  // unrolled
#pragma unroll
                    for (uint32_t p = 0; p < 3u; ++p) {
                        if (p >= np) break;
                        const uint32_t pl = __ballot_sync(0xffffffffu, (cls[u] >> p) & 1u);
                        if (lane == p) word = pl;
                    }
#pragma unroll
                    for (uint32_t j = 1; j <= (uint32_t)NJ; ++j) {
                        const uint32_t bj = __ballot_sync(0xffffffffu, cls[u] == j);
                        if (lane == j - 1) ccount[(uint64_t)(j - 1) * nblk + blk] = __popc(bj);
                    }
                } else {
#pragma unroll 1
                    for (uint32_t p = 0; p < np; ++p) {
                        const uint32_t pl = __ballot_sync(0xffffffffu, (cls[u] >> p) & 1u);
                        if (lane == p) word = pl;
                    }
#pragma unroll 1
                    for (uint32_t j = 1; j <= J; ++j) {
                        const uint32_t bj = __ballot_sync(0xffffffffu, cls[u] == j);
                        if (lane == j - 1) ccount[(uint64_t)(j - 1) * nblk + blk] = __popc(bj);
                    }
                }
                if (lane < np) rec[(rec0 + bi) * Rp + lane] = word;
            }
        }
    }
}

__global__ void rec_fill_kernel(const uint64_t* __restrict__ cpre, uint64_t nblk, uint32_t np,
                                uint32_t J, uint32_t Rp, uint32_t* __restrict__ rec, uint32_t nloc,
                                uint32_t E, uint32_t MB) {
    for (uint64_t x = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; x < nblk * J;
         x += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t blk = x / J;  // worker-major block order of the prefix scan
        const uint32_t j = (uint32_t)(x % J);
        const uint64_t seg = blk / MB;
        const uint32_t wl = (uint32_t)(seg / E), e = (uint32_t)(seg - (uint64_t)wl * E);
        rec[rec_index(wl, e, nloc, MB, (uint32_t)(blk - seg * MB)) * Rp + np + j] =
            (uint32_t)cpre[(uint64_t)j * (nblk + 1) + blk];
    }
}

// class base of every (worker, class): prefix count at the worker's first block
__global__ void class_base_kernel(const uint64_t* __restrict__ cpre, uint64_t nblk, uint32_t nloc,
                                  uint32_t E, uint32_t MB, uint32_t J, uint32_t* __restrict__ cbase) {
    for (uint32_t x = blockIdx.x * blockDim.x + threadIdx.x; x < nloc * J; x += gridDim.x * blockDim.x) {
        const uint32_t wl = x / J, j = x % J;
        cbase[x] = (uint32_t)cpre[(uint64_t)j * (nblk + 1) + (uint64_t)wl * E * MB];
    }
}

// class_list[cstart[wl*J + j-1] + pos] = sample, pos = position in the worker's class list.
// One warp per (worker, epoch) segment, kBU blocks per iteration; the block record is spread
// over lanes 0..Rp-1 and read through shuffles, the stream words are loaded up front.
template <int NP>  // class bit-planes (0: runtime np)
__global__ void __launch_bounds__(kThreads) class_write_kernel(
    Part part, uint32_t MB, const uint32_t* __restrict__ stream, const uint32_t* __restrict__ rec,
    uint32_t np_rt, uint32_t J, uint32_t Rp, const uint32_t* __restrict__ cbase,
    const uint64_t* __restrict__ cstart, uint32_t* __restrict__ class_list, uint64_t nblk) {
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t np = NP > 0 ? (uint32_t)NP : np_rt;
    const uint32_t E = part.E, nloc = part.wend - part.wbegin;
    const uint64_t nseg = (uint64_t)nloc * E;
    for (uint64_t seg = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; seg < nseg;
         seg += ((uint64_t)gridDim.x * blockDim.x) >> 5) {
        const uint32_t wl = (uint32_t)(seg / E), e = (uint32_t)(seg - (uint64_t)wl * E);
        const uint32_t w = part.wbegin + wl;
        const uint64_t Le = part.epoch_len(w);
        const uint64_t g0 = part.stream_offset(w) + (uint64_t)e * Le;
        const uint64_t blk0 = rec_index(wl, e, nloc, MB, 0);
        // class bases / list starts of this worker: lanes j < J
        const uint32_t cb = lane < J ? cbase[wl * J + lane] : 0;
        const uint64_t cs = lane < J ? cstart[(uint64_t)wl * J + lane] : 0;
        const uint32_t nb = (uint32_t)((Le + 31) >> 5);
        for (uint32_t b0 = 0; b0 < nb; b0 += kBU) {
            uint32_t mine[kBU], kv[kBU];
#pragma unroll
            for (int u = 0; u < kBU; ++u) {
                const uint32_t bi = b0 + u;
                const uint64_t t = (uint64_t)bi * 32 + lane;
                mine[u] = (bi < nb && lane < Rp) ? rec[(blk0 + bi) * Rp + lane] : 0;
                kv[u] = (bi < nb && t < Le) ? __ldcs(stream + g0 + t) : 0;
            }
#pragma unroll
            for (int u = 0; u < kBU; ++u) {
                const uint32_t bi = b0 + u;
                if (bi >= nb) break;
                const uint64_t t = (uint64_t)bi * 32 + lane;
                uint32_t cls = 0, cm = 0xffffffffu;
#pragma unroll
                for (uint32_t p = 0; p < (NP > 0 ? (uint32_t)NP : 8u); ++p) {
                    if (p >= np) break;
                    cls |= ((__shfl_sync(0xffffffffu, mine[u], p) >> lane) & 1u) << p;
                }
                if (t >= Le) cls = 0;
#pragma unroll
                for (uint32_t p = 0; p < (NP > 0 ? (uint32_t)NP : 8u); ++p) {
                    if (p >= np) break;
                    const uint32_t pl = __shfl_sync(0xffffffffu, mine[u], p);
                    cm &= ((cls >> p) & 1u) ? pl : ~pl;
                }
                const uint32_t ci = cls ? cls - 1 : 0;
                const uint32_t pre = __shfl_sync(0xffffffffu, mine[u], (np + ci) & 31);
                const uint32_t base = __shfl_sync(0xffffffffu, cb, ci & 31);
                const uint64_t start = __shfl_sync(0xffffffffu, cs, ci & 31);
                if (cls) __stcs(class_list + start + (pre - base) + __popc(cm & lanemask_lt()), kv[u]);
            }
        }
    }
}

// per (worker, class) list lengths from the class prefix counts
__global__ void class_lens_kernel(uint32_t nloc, uint32_t E, uint32_t MB, uint32_t J,
                                  const uint64_t* __restrict__ cpre, uint64_t nblk,
                                  uint64_t* __restrict__ clen) {
    for (uint32_t x = blockIdx.x * blockDim.x + threadIdx.x; x < nloc * J; x += gridDim.x * blockDim.x) {
        const uint32_t wl = x / J, j = x % J;
        const uint64_t a = (uint64_t)wl * E * MB, b = (uint64_t)(wl + 1) * E * MB;
        clen[x] = cpre[(uint64_t)j * (nblk + 1) + b] - cpre[(uint64_t)j * (nblk + 1) + a];
    }
}

// ---------------------------------------------------------------------------- K8
// One CTA takes 32 samples: their inverse-permutation and rank rows are loaded with coalesced
// 128-B rows into padded shared tiles; then one warp per sample, lanes = epochs: every first
// access (rank != 0xFFFF) looks up its class and class-list position in the block record and
// writes its holder record {worker, class, position} at pair_off[k] + rank (build_index
// order, workers ascending): a warp's stores land in one sample's contiguous holder range.
// (Measured slower for config 2 and dropped: staging the records in shared memory for fully
// contiguous stores — MIO-throttled, 2.2 vs 1.15 ms — 4 samples per warp in flight with
// double-buffered cp.async tiles — register-limited occupancy, 1.5-1.7 ms — and the cp.async
// double buffer alone, 1.13 vs 1.05 ms.)
// NP: class bit-planes per record (0: runtime np); NP == -1: all-fit records (uint2 {first
// mask, class-1 prefix}, every first access is class 1).
__device__ __forceinline__ uint32_t pick(const uint4& a, uint32_t i) {
    return i == 0 ? a.x : i == 1 ? a.y : i == 2 ? a.z : a.w;
}

__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
    const uint32_t s = (uint32_t)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

template <int NP, int TU = 4>  // TU: tile rows in flight per thread (8 spills: slower)
__global__ void __launch_bounds__(kThreads, 5) holder_tile_kernel(
    Part part, const uint32_t* __restrict__ inv, const uint16_t* __restrict__ rank16, uint32_t MB,
    const uint32_t* __restrict__ rec, uint32_t np_rt, uint32_t J, uint32_t Rp,
    const uint32_t* __restrict__ cbase, const uint64_t* __restrict__ pair_off,
    uint32_t* __restrict__ holders, const uint32_t* __restrict__ gate) {
    if (gate && *gate == 0) return;  // speculative all-fit launch, the test failed
    extern __shared__ uint32_t sm[];
    const uint32_t E = part.E, F = part.F;
    const uint32_t np = NP > 0 ? (uint32_t)NP : np_rt;
    uint32_t* tinv = sm;                                            // [E][33]
    uint16_t* trk = reinterpret_cast<uint16_t*>(sm + (size_t)E * 33);  // [E][33]
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
    for (uint64_t k0 = (uint64_t)blockIdx.x * 32; k0 < F; k0 += (uint64_t)gridDim.x * 32) {
        __syncthreads();
        for (uint32_t i0 = threadIdx.x; i0 < E * 32; i0 += TU * blockDim.x) {
            uint32_t iv[TU];
            uint16_t rv[TU];
#pragma unroll
            for (int u = 0; u < TU; ++u) {
                const uint32_t idx = i0 + u * blockDim.x;
                const uint32_t e = idx >> 5, l = idx & 31;
                const bool ok = idx < E * 32 && k0 + l < F;
                iv[u] = ok ? __ldcs(inv + (size_t)e * part.Fp + k0 + l) : kNone;
                rv[u] = ok ? __ldcs(rank16 + (size_t)e * part.Fp + k0 + l) : (uint16_t)0xFFFFu;
            }
#pragma unroll
            for (int u = 0; u < TU; ++u) {
                const uint32_t idx = i0 + u * blockDim.x;
                if (idx < E * 32) {
                    const uint32_t e = idx >> 5, l = idx & 31;
                    tinv[e * 33 + l] = iv[u];
                    trk[e * 33 + l] = rv[u];
                }
            }
        }
        __syncthreads();
        if constexpr (NP == -1) {
            if (E <= 128) {  // all-fit, <= 4 epoch rounds: the rounds' record loads overlap
                for (uint32_t s = warp; s < 32; s += nwarps) {
                    if (k0 + s >= F) break;
                    const uint64_t slot0 = pair_off[k0 + s];
                    uint32_t rk[4], w[4], bit[4];
                    uint2 a2[4];
                    uint32_t cb[4];
#pragma unroll
                    for (int r = 0; r < 4; ++r) {
                        const uint32_t e = r * 32 + lane;
                        rk[r] = e < E ? trk[e * 33 + s] : 0xFFFFu;
                        if (rk[r] != 0xFFFFu) {
                            const uint32_t tseg = part.within_epoch(tinv[e * 33 + s], w[r]);
                            const uint32_t wl = w[r] - part.wbegin;
                            const uint64_t blk = rec_index(wl, e, part.wend - part.wbegin, MB, tseg >> 5);
                            bit[r] = tseg & 31;
                            a2[r] = __ldg(reinterpret_cast<const uint2*>(rec) + blk);
                            cb[r] = __ldg(cbase + wl * J);
                        }
                    }
#pragma unroll
                    for (int r = 0; r < 4; ++r) {
                        if (rk[r] == 0xFFFFu) continue;
                        const uint32_t cls = (a2[r].x >> bit[r]) & 1u;
                        const uint32_t pos =
                            cls ? a2[r].y - cb[r] + __popc(a2[r].x & ((1u << bit[r]) - 1u)) : 0u;
                        uint32_t* h = holders + 3 * (slot0 + rk[r]);
                        __stcs(h, w[r]);
                        __stcs(h + 1, cls);
                        __stcs(h + 2, pos);
                    }
                }
                continue;
            }
        }
        for (uint32_t s = warp; s < 32; s += nwarps) {
            if (k0 + s >= F) break;
            const uint64_t slot0 = pair_off[k0 + s];
            for (uint32_t e = lane; e < E; e += 32) {
                const uint32_t rk = trk[e * 33 + s];
                if (rk == 0xFFFFu) continue;
                uint32_t w;
                const uint32_t tseg = part.within_epoch(tinv[e * 33 + s], w);
                const uint32_t wl = w - part.wbegin;
                const uint64_t blk = rec_index(wl, e, part.wend - part.wbegin, MB, tseg >> 5);
                const uint32_t bit = tseg & 31;
                uint32_t cls, pos = 0;
                if constexpr (NP == -1) {
                    // one 64-bit load and the class base issued together (a plain uint2 read
                    // was split into two dependent 32-bit loads)
                    const uint2 a2 = __ldg(reinterpret_cast<const uint2*>(rec) + blk);
                    const uint32_t cb = __ldg(cbase + wl * J);
                    cls = (a2.x >> bit) & 1u;
                    pos = cls ? a2.y - cb + __popc(a2.x & ((1u << bit) - 1u)) : 0u;
                } else {
                const uint4 a = __ldg(reinterpret_cast<const uint4*>(rec + blk * Rp));
                uint32_t cb0 = 0, cb1 = 0, cb2 = 0;  // class bases issued with the record (J <= 3)
                if constexpr (NP == 1 || NP == 2) {
                    cb0 = __ldg(cbase + wl * J);
                    if (J > 1) cb1 = __ldg(cbase + wl * J + 1);
                    if (J > 2) cb2 = __ldg(cbase + wl * J + 2);
                }
                uint32_t cm;
                if constexpr (NP == 1) {
                    cls = (a.x >> bit) & 1u;
                    cm = a.x;
                } else if constexpr (NP == 2) {
                    const uint32_t b0 = (a.x >> bit) & 1u, b1 = (a.y >> bit) & 1u;
                    cls = b0 | (b1 << 1);
                    cm = (b0 ? a.x : ~a.x) & (b1 ? a.y : ~a.y);
                } else {
                    cls = 0;
                    for (uint32_t q = 0; q < np; ++q) cls |= ((pick(a, q) >> bit) & 1u) << q;
                    cm = 0xffffffffu;
                    for (uint32_t q = 0; q < np; ++q) {
                        const uint32_t pl = pick(a, q);
                        cm &= ((cls >> q) & 1u) ? pl : ~pl;
                    }
                }
                if (cls) {
                    const uint32_t wi = np + cls - 1;
                    const uint32_t prew = wi < 4 ? pick(a, wi) : rec[blk * Rp + wi];
                    uint32_t cb;
                    if constexpr (NP == 1 || NP == 2) cb = cls == 1 ? cb0 : cls == 2 ? cb1 : cb2;
                    else cb = cbase[wl * J + cls - 1];
                    pos = prew - cb + __popc(cm & ((1u << bit) - 1u));
                }
                }
                uint32_t* h = holders + 3 * (slot0 + rk);
                __stcs(h, w);
                __stcs(h + 1, cls);
                __stcs(h + 2, pos);
            }
        }
    }
}

// ---------------------------------------------------------------------------- K4a (tile)
// CTA = 32 samples: the tile inv[0..E)[k0..k0+32) arrives in shared memory by double-buffered
// cp.async; one warp per sample, lanes = epochs (R rounds of 32).  Per-warp shared tables
// indexed by local worker — first epoch (atomicMin), access count (atomicAdd) and a worker
// bitmap (atomicOr) — give every pair's count and first access; the bitmap's popcount prefix
// is the pair's rank (build_index worker order).  info / rank rows go back through a shared
// output tile with coalesced stores.  Needs nloc <= kTileWorkers, E <= 32 R.
constexpr uint32_t kTileWorkers = 1024;
constexpr uint32_t kStInv = 33, kStOut = 34;

__device__ __forceinline__ void st_issue(const uint32_t* inv, uint32_t E, uint32_t F, uint64_t k0,
                                         uint32_t* tinv) {
    const uint32_t n = (uint32_t)(F - k0 < 32 ? F - k0 : 32);
    for (uint32_t idx = threadIdx.x; idx < E * 32; idx += blockDim.x) {
        const uint32_t e = idx >> 5, l = idx & 31;
        if (l < n) cp_async4(tinv + e * kStInv + l, inv + (size_t)e * pitch16(F) + k0 + l);
    }
    cp_async_commit();
}

template <int R, typename IT>
__global__ void __launch_bounds__(kThreads) sample_tile_kernel(Part part, const uint32_t* __restrict__ inv,
                                                               IT* __restrict__ info,
                                                               uint16_t* __restrict__ rank16,
                                                               uint32_t* __restrict__ pair_count,
                                                               uint32_t W,
                                                               uint32_t* __restrict__ seghist,
                                                               WorkerSums ws) {
    extern __shared__ uint32_t sm[];
    const uint32_t E = part.E, F = part.F;
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
    const uint32_t nloc = part.wend - part.wbegin;
    uint32_t* tin[2] = {sm, sm + E * kStInv};
    uint16_t* orank = reinterpret_cast<uint16_t*>(sm + 2 * E * kStInv);  // [E][34]
    IT* oinfo = reinterpret_cast<IT*>(orank + E * kStOut);                 // [E][kSI]
    constexpr uint32_t kSI = sizeof(IT) == 1 ? 36 : kStOut;  // row stride: 4-B aligned rows
    uint32_t* tabs = sm + 2 * E * kStInv + E * kStOut;                    // per warp
    uint32_t* fe = tabs + warp * (2 * W * 32 + W);  // [nloc] first epoch
    uint32_t* cnt = fe + W * 32;                     // [nloc] count
    uint32_t* bm = cnt + W * 32;                     // [W] worker bitmap
    // per-CTA candidate size sums / counts per local worker (the whole-worker fit test)
    // (fixed point, size * 2^20 rounded up: an upper bound; 64-bit sums as two 32-bit words,
    // native shared atomics)
    uint32_t* clo = tabs + nwarps * (2 * W * 32 + W);
    uint32_t* chi = clo + W * 32;
    uint32_t* ccnt = chi + W * 32;
    if (ws.sum)
        for (uint32_t x = threadIdx.x; x < W * 32; x += blockDim.x) {
            clo[x] = 0;
            chi[x] = 0;
            ccnt[x] = 0;
        }
    for (uint32_t x = lane; x < W * 32; x += 32) {
        fe[x] = kNone;
        cnt[x] = 0;
    }
    if (lane < W) bm[lane] = 0;
    __syncthreads();
    const uint64_t stride = (uint64_t)gridDim.x * 32;
    uint64_t k0 = (uint64_t)blockIdx.x * 32;
    if (k0 < F) st_issue(inv, E, F, k0, tin[0]);
    for (uint32_t buf = 0; k0 < F; k0 += stride, buf ^= 1) {
        if (k0 + stride < F) {
            st_issue(inv, E, F, k0 + stride, tin[buf ^ 1]);
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncthreads();
        const uint32_t* tinv = tin[buf];
        for (uint32_t s = warp; s < 32; s += nwarps) {
            const bool live = k0 + s < F;
            // the sample's size, issued early (used after the rounds)
            const double szv = (ws.sum && live) ? __ldg(ws.sizes + k0 + s) : 0.0;
            uint32_t wl[R];
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const uint32_t e = r * 32 + lane;
                wl[r] = kNone;
                if (live && e < E) {
                    const uint32_t p = tinv[e * kStInv + s];
                    if (p < part.P) {
                        const uint32_t w = part.worker_of(p);
                        if (w >= part.wbegin && w < part.wend) {
                            const uint32_t x = w - part.wbegin;
                            wl[r] = x;
                            atomicMin(&fe[x], e);
                            atomicAdd(&cnt[x], 1u);
                            atomicOr(&bm[x >> 5], 1u << (x & 31));
                        }
                    }
                }
            }
            __syncwarp();
            // exclusive popcount prefix of the bitmap words: lane t holds word t
            const uint32_t word = lane < W ? bm[lane] : 0u;
            const uint32_t c = __popc(word);
            uint32_t inc = c;
#pragma unroll
            for (uint32_t d = 1; d < 32; d <<= 1) {  // lanes >= W hold 0 (fixed 5 steps, no loop)
                const uint32_t o = __shfl_up_sync(0xffffffffu, inc, d);
                if (lane >= d) inc += o;
            }
            const uint32_t pre = inc - c;
            const uint32_t total = __shfl_sync(0xffffffffu, inc, W - 1);
            if (live && lane == 0) pair_count[k0 + s] = total;
            unsigned long long sz = 0;
            if (ws.sum && live) {
                const double v = szv;
                if (!(v >= 0.0 && v < 0x1.0p40)) {
                    if (lane == 0) atomicOr(ws.neg, 1u);  // negative, NaN or huge: no all-fit
                } else {
                    sz = __double2ull_ru(v * 0x1.0p20);
                }
            }
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const uint32_t e = r * 32 + lane;
                const uint32_t x = wl[r];
                const uint32_t xw = x != kNone ? x >> 5 : 0u;
                const uint32_t pw = __shfl_sync(0xffffffffu, pre, xw);
                const uint32_t ww = __shfl_sync(0xffffffffu, word, xw);
                if (e < E) {
                    IT ci = 0;
                    uint16_t rk = 0xFFFFu;
                    if (x != kNone && fe[x] == e) {
                        ci = (IT)cnt[x];
                        rk = (uint16_t)(pw + __popc(ww & ((1u << (x & 31)) - 1u)));
                        if (seghist) atomicAdd(&seghist[((uint64_t)x * E + (E - ci)) * E + e], 1u);
                        if (ws.sum) {
                            add64(clo + x, chi + x, sz);
                            atomicAdd(&ccnt[x], 1u);
                        }
                    }
                    oinfo[e * kSI + s] = ci;
                    orank[e * kStOut + s] = rk;
                }
            }
            __syncwarp();
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const uint32_t x = wl[r];
                if (x != kNone) {
                    fe[x] = kNone;
                    cnt[x] = 0;
                }
            }
            if (lane < W) bm[lane] = 0;
            __syncwarp();
        }
        __syncthreads();
        // coalesced write-back of the info / rank rows: 16-B stores of 16 / 8 samples (the
        // rows are pitched to Fp, a multiple of 16 samples), scalar for a partial last tile
        const uint32_t n = (uint32_t)(F - k0 < 32 ? F - k0 : 32);
        if (n == 32) {
            constexpr uint32_t IQ = 16 / sizeof(IT);  // samples per 16-B info store
            for (uint32_t idx = threadIdx.x; idx < E * 4; idx += blockDim.x) {
                const uint32_t e = idx >> 2, q = (idx & 3) * 8;
                const uint32_t* sr = reinterpret_cast<const uint32_t*>(orank + e * kStOut + q);
                __stcs(reinterpret_cast<uint4*>(rank16 + (size_t)e * part.Fp + k0 + q),
                       make_uint4(sr[0], sr[1], sr[2], sr[3]));
            }
            for (uint32_t idx = threadIdx.x; idx < E * (32 / IQ); idx += blockDim.x) {
                const uint32_t e = idx / (32 / IQ), q = (idx % (32 / IQ)) * IQ;
                const uint32_t* si = reinterpret_cast<const uint32_t*>(oinfo + e * kSI + q);
                __stcs(reinterpret_cast<uint4*>(info + (size_t)e * part.Fp + k0 + q),
                       make_uint4(si[0], si[1], si[2], si[3]));
            }
        } else {
            for (uint32_t idx = threadIdx.x; idx < E * 32; idx += blockDim.x) {
                const uint32_t e = idx >> 5, l = idx & 31;
                if (l < n) {
                    __stcs(info + (size_t)e * part.Fp + k0 + l, oinfo[e * kSI + l]);
                    __stcs(rank16 + (size_t)e * part.Fp + k0 + l, orank[e * kStOut + l]);
                }
            }
        }
        // the output tile and the input buffer are reused after the next barrier
    }
    if (ws.sum) {
        __syncthreads();
        for (uint32_t x = threadIdx.x; x < nloc; x += blockDim.x) {
            if (ccnt[x]) {
                atomicAdd(&ws.sum[x], ((unsigned long long)chi[x] << 32) | clo[x]);
                atomicAdd(&ws.cnt[x], ccnt[x]);
            }
        }
    }
}

// ---------------------------------------------------------------------------- launchers
constexpr uint32_t kMaxLaneWorkers = 2048;

bool lane_path_ok(const Part& part) {
    // per-lane shared rows: 2 x W bitmap words + E x (worker, count) u16 pairs, 4 warps / CTA
    return (part.wend - part.wbegin) <= kMaxLaneWorkers && part.E <= 1024;
}

void launch_blk_codes(cudaStream_t s, const Part& part, uint32_t MB, const uint32_t* blkmask,
                      const uint32_t* blkbase, const uint32_t* dest, const uint8_t* cls_sorted,
                      uint32_t np, uint32_t J, uint32_t Rp, uint32_t* rec, uint32_t* ccount,
                      uint64_t nblk) {
    const uint64_t nseg = (uint64_t)(part.wend - part.wbegin) * part.E;
    const unsigned g = grid_for(nseg * 32, kThreads, 148u * 64u);
    if (J == 1)
        blk_codes_kernel<1><<<g, kThreads, 0, s>>>(part, MB, blkmask, blkbase, dest, cls_sorted, np, J, Rp, rec, ccount, nblk);
    else if (J == 2)
        blk_codes_kernel<2><<<g, kThreads, 0, s>>>(part, MB, blkmask, blkbase, dest, cls_sorted, np, J, Rp, rec, ccount, nblk);
    else if (J == 3)
        blk_codes_kernel<3><<<g, kThreads, 0, s>>>(part, MB, blkmask, blkbase, dest, cls_sorted, np, J, Rp, rec, ccount, nblk);
    else
        blk_codes_kernel<0><<<g, kThreads, 0, s>>>(part, MB, blkmask, blkbase, dest, cls_sorted, np, J, Rp, rec, ccount, nblk);
}

void launch_rec_fill(cudaStream_t s, const uint64_t* cpre, uint64_t nblk, uint32_t np, uint32_t J,
                     uint32_t Rp, uint32_t* rec, uint32_t nloc, uint32_t E, uint32_t MB,
                     uint32_t* cbase) {
    rec_fill_kernel<<<grid_for(nblk * J, kThreads), kThreads, 0, s>>>(cpre, nblk, np, J, Rp, rec, nloc, E,
                                                                     MB);
    class_base_kernel<<<grid_for((uint64_t)nloc * J, kThreads), kThreads, 0, s>>>(cpre, nblk, nloc, E,
                                                                                 MB, J, cbase);
}

void launch_class_write(cudaStream_t s, const Part& part, uint32_t MB, const uint32_t* stream,
                        const uint32_t* rec, uint32_t np, uint32_t J, uint32_t Rp,
                        const uint32_t* cbase, const uint64_t* cstart, uint32_t* class_list,
                        uint64_t nblk) {
    const uint64_t nseg = (uint64_t)(part.wend - part.wbegin) * part.E;
    const unsigned g = grid_for(nseg * 32, kThreads, 148u * 64u);
    if (np == 1)
        class_write_kernel<1><<<g, kThreads, 0, s>>>(part, MB, stream, rec, np, J, Rp, cbase, cstart, class_list, nblk);
    else if (np == 2)
        class_write_kernel<2><<<g, kThreads, 0, s>>>(part, MB, stream, rec, np, J, Rp, cbase, cstart, class_list, nblk);
    else
        class_write_kernel<0><<<g, kThreads, 0, s>>>(part, MB, stream, rec, np, J, Rp, cbase, cstart, class_list, nblk);
}

void launch_class_lens(cudaStream_t s, uint32_t nloc, uint32_t E, uint32_t MB, uint32_t J,
                       const uint64_t* cpre, uint64_t nblk, uint64_t* clen) {
    class_lens_kernel<<<grid_for((uint64_t)nloc * J, kThreads), kThreads, 0, s>>>(nloc, E, MB, J, cpre,
                                                                                 nblk, clen);
}

void launch_holder_tile(cudaStream_t s, const Part& part, const uint32_t* inv, const uint16_t* rank16,
                        uint32_t MB, const uint32_t* rec, uint32_t np, uint32_t J, uint32_t Rp,
                        const uint32_t* cbase, const uint64_t* pair_off, uint32_t* holders,
                        bool allfit, const uint32_t* gate) {
    const size_t smem = (size_t)part.E * 33 * 4 + (size_t)part.E * 33 * 2 + 16;
    const uint64_t tiles = ((uint64_t)part.F + 31) / 32;
    // CTAs per SM in the grid (config 2: 10 -> 1.088, 16 -> 1.116, 5 -> 1.097 ms)
    static const int gmul = (int)ab_knob("CLAIRPLAN_HOLDER_GRID", 10);
    const unsigned grid = grid_for(tiles, 1, 148u * (unsigned)gmul);
#define HT_LAUNCH(NPV)                                                                           \
    do {                                                                                         \
        allow_smem(holder_tile_kernel<NPV>, \
                             (int)smem);                                                         \
        holder_tile_kernel<NPV><<<grid, kThreads, smem, s>>>(part, inv, rank16, MB, rec, np, J, Rp, \
                                                             cbase, pair_off, holders, gate);    \
    } while (0)
    if (allfit) HT_LAUNCH(-1);
    else if (np == 1) HT_LAUNCH(1);
    else if (np == 2) HT_LAUNCH(2);
    else HT_LAUNCH(0);
#undef HT_LAUNCH
}

void launch_sample_lanes(cudaStream_t s, const Part& part, const uint32_t* inv, uint16_t* info,
                         uint16_t* rank16, uint32_t* pair_count, uint32_t* seghist) {
    const uint32_t nloc = part.wend - part.wbegin;
    const uint32_t W = (nloc + 31) / 32;
    const size_t smem = (size_t)4 * (64 * W + 32 * part.E) * 4;
    allow_smem(sample_lanes_kernel, (int)smem);
    const uint64_t groups = ((uint64_t)part.F + 31) / 32;
    sample_lanes_kernel<<<grid_for(groups, 4, 148u * 8u), 128, smem, s>>>(part, inv, info, rank16,
                                                                         pair_count, W, seghist);
}

bool tile_path_ok(const Part& part) {
    return (part.wend - part.wbegin) <= kTileWorkers && part.E <= 128;
}

void launch_sample_tile(cudaStream_t s, const Part& part, const uint32_t* inv, void* info, bool info8,
                        uint16_t* rank16, uint32_t* pair_count, uint32_t* seghist,
                        const WorkerSums& ws) {
    const uint32_t nloc = part.wend - part.wbegin;
    const uint32_t W = (nloc + 31) / 32;
    const size_t smem = (size_t)4 * (2 * part.E * kStInv + part.E * kStOut +
                                     (kThreads / 32) * (2 * W * 32 + W) + 2) +
                        (ws.sum ? (size_t)W * 32 * 12 : 0);  // clo, chi, ccnt
    const uint64_t tiles = ((uint64_t)part.F + 31) / 32;
    static const unsigned gm = ab_knob("CLAIRPLAN_GRID_SAMPLE", 16);
    const unsigned grid = grid_for(tiles, 1, 148u * gm);
#define ST_LAUNCH(RV)                                                                             \
    do {                                                                                          \
        if (info8) {                                                                              \
            allow_smem(sample_tile_kernel<RV, uint8_t>,                                 \
                                 (int)smem);         \
            sample_tile_kernel<RV, uint8_t><<<grid, kThreads, smem, s>>>(                         \
                part, inv, static_cast<uint8_t*>(info), rank16, pair_count, W, seghist, ws);      \
        } else {                                                                                  \
            allow_smem(sample_tile_kernel<RV, uint16_t>,                                \
                                 (int)smem);         \
            sample_tile_kernel<RV, uint16_t><<<grid, kThreads, smem, s>>>(                        \
                part, inv, static_cast<uint16_t*>(info), rank16, pair_count, W, seghist, ws);     \
        }                                                                                         \
    } while (0)
    const uint32_t R = (part.E + 31) / 32;
    if (R == 1) ST_LAUNCH(1);
    else if (R == 2) ST_LAUNCH(2);
    else if (R == 3) ST_LAUNCH(3);
    else ST_LAUNCH(4);
#undef ST_LAUNCH
}

void launch_sample_hash(cudaStream_t s, const Part& part, const uint32_t* inv, uint16_t* info,
                        uint16_t* rank16, uint32_t* pair_count, const uint32_t* list,
                        const uint32_t* nlist, uint64_t max_items, uint32_t* seghist) {
    const uint32_t nloc = part.wend - part.wbegin;
    const uint32_t d = part.E < nloc ? part.E : nloc;
    uint32_t hs = 32;
    while (hs < 2 * d) hs <<= 1;
    const uint32_t W = (nloc + 31) / 32;
    const size_t smem = (size_t)4 * (2 * hs + 2 * W) * 4;
    allow_smem(sample_hash_kernel, (int)smem);
    sample_hash_kernel<<<grid_for(max_items, 4, 148u * 16u), 128, smem, s>>>(
        part, inv, info, rank16, pair_count, list, nlist, hs, W, seghist);
}

void launch_seg_hist(cudaStream_t s, const Part& part, const uint32_t* stream, const void* info,
                     bool info8, const uint32_t* cpos, uint32_t* seghist, uint32_t* segcnt) {
    const uint64_t nseg = (uint64_t)(part.wend - part.wbegin) * part.E;
    const size_t smem = (size_t)(kThreads / 32) * part.E * 4;
    const unsigned grid = grid_for(nseg * 32, kThreads, 148u * 64u);
    if (info8) {
        allow_smem(seg_hist_kernel<uint8_t>, (int)smem);
        seg_hist_kernel<uint8_t><<<grid, kThreads, smem, s>>>(part, stream, static_cast<const uint8_t*>(info),
                                                              cpos, seghist, segcnt);
    } else {
        allow_smem(seg_hist_kernel<uint16_t>, (int)smem);
        seg_hist_kernel<uint16_t><<<grid, kThreads, smem, s>>>(part, stream, static_cast<const uint16_t*>(info),
                                                               cpos, seghist, segcnt);
    }
}


void launch_seg_write2(cudaStream_t s, const Part& part, const uint32_t* stream, const uint16_t* info, const uint32_t* cpos,
                       const double* sizes, const uint64_t* seg_off, const uint64_t* sorted_base,
                       uint32_t MB, uint32_t* dest, double* sorted_size, uint32_t* blkmask,
                       uint32_t* blkbase) {
    const uint64_t nseg = (uint64_t)(part.wend - part.wbegin) * part.E;
    const size_t smem = (size_t)(kThreads / 32) * part.E * 4;
    allow_smem(seg_write_kernel2<uint16_t>, (int)smem);
    seg_write_kernel2<uint16_t><<<grid_for(nseg * 32, kThreads, 148u * 64u), kThreads, smem, s>>>(
        part, stream, info, cpos, sizes, seg_off, sorted_base, MB, dest, sorted_size, blkmask, blkbase);
}

}  // namespace clairplan
