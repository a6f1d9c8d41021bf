// Sparse sample-major passes of a worker-sharded handle (multi-GPU).
//
// A rank holds 1/G of the stream entries; the dense [E][F] sample-major arrays of the
// single-GPU path (inv, info, rank) would cost E*F work on every rank.  Instead:
//   csr_hist / csr_scatter   counting sort of the local stream entries by sample
//                            (csr[koff[k] ..] = stream indices of sample k)
//   sparse_sample            warp per sample over its entries: per local worker the first
//                            access (smallest stream index = earliest epoch, access.cpp:59-78
//                            order), the access count, the worker bitmap -> pair_count[k],
//                            einfo[slot] = count at a pair's first access (0 elsewhere) and
//                            erank[slot] = the pair's rank among the sample's local workers
//                            (build_index worker order, policies.cpp:124-142), in CSR order;
//                            cpos[s] (stream index -> CSR slot) lets the segment passes find
//                            an entry's value
//   holder_sparse            thread per CSR entry: holder records at pair_off[k] + rank from
//                            the block records of the tier / all-fit paths
// The CSR is written in sample windows that fit L2 (the random slot writes then merge there).
#include <cstdlib>

#include "internal.h"

namespace clairplan {

// local worker of stream index s: largest wl with soff[wl] <= s (soff[nloc] = total); when
// every local worker's stream has the same length (FastDiv d != 1 ... set by the host), one
// division
__device__ __forceinline__ uint32_t worker_of_entry(const uint64_t* __restrict__ soff, uint32_t nloc,
                                                    uint64_t s, const FastDiv& uni) {
    if (uni.d > 1 || nloc == 1) return nloc == 1 ? 0u : uni.div((uint32_t)s);
    uint32_t lo = 0, hi = nloc;
    while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if (__ldg(soff + mid) <= s) lo = mid;
        else hi = mid;
    }
    return lo;
}

__global__ void __launch_bounds__(kThreads) csr_hist_kernel(const uint32_t* __restrict__ stream,
                                                            uint64_t n, uint32_t* __restrict__ cnt) {
    for (uint64_t s = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; s < n;
         s += (uint64_t)gridDim.x * blockDim.x)
        atomicAdd(&cnt[__ldcs(stream + s)], 1u);
}

__global__ void __launch_bounds__(kThreads) csr_cursor_kernel(const uint64_t* __restrict__ koff,
                                                              uint32_t F, uint32_t* __restrict__ cur) {
    for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < F; k += gridDim.x * blockDim.x)
        cur[k] = (uint32_t)koff[k];
}

// entries whose sample lies in [k_lo, k_hi) (a window of the CSR that stays L2-resident while
// it is written): csr[slot] = s, cpos[s] = slot
__global__ void __launch_bounds__(kThreads) csr_scatter_kernel(const uint32_t* __restrict__ stream,
                                                               uint64_t n, uint32_t k_lo, uint32_t k_hi,
                                                               uint32_t* __restrict__ cur,
                                                               uint32_t* __restrict__ csr,
                                                               uint32_t* __restrict__ cpos) {
    // 4 entries per thread and round: their cursor atomics are independent and overlap
    constexpr int U = 4;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t s0 = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; s0 < n; s0 += U * stride) {
        uint32_t k[U], slot[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint64_t s = s0 + u * stride;
            k[u] = s < n ? __ldcs(stream + s) : kNone;
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
            slot[u] = (k[u] >= k_lo && k[u] < k_hi) ? atomicAdd(&cur[k[u]], 1u) : kNone;
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (slot[u] == kNone) continue;
            const uint64_t s = s0 + u * stride;
            csr[slot[u]] = (uint32_t)s;
            cpos[s] = slot[u];
        }
    }
}

// warp per sample, lanes over its entries (R rounds of 32, entries kept in registers); per-warp
// shared tables indexed by local worker (nloc <= 32 W)
template <int R>
__global__ void __launch_bounds__(kThreads, 5) sparse_sample_kernel(
    uint32_t F, uint32_t nloc, uint32_t W, const uint64_t* __restrict__ soff,
    const uint64_t* __restrict__ koff, const uint32_t* __restrict__ csr,
    uint32_t* __restrict__ pair_count, uint16_t* __restrict__ einfo, uint16_t* __restrict__ erank,
    WorkerSums ws, FastDiv uni) {
    extern __shared__ uint32_t sm[];
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    constexpr uint32_t NW = kThreads / 32;
    uint32_t* fs = sm + warp * (2 * W * 32 + W);  // [nloc] smallest stream index
    uint32_t* cnt = fs + W * 32;                   // [nloc] accesses
    uint32_t* bm = cnt + W * 32;                   // [W]
    // per-CTA candidate size sums / counts per local worker (the whole-worker fit test)
    // (fixed point, size * 2^20 rounded up: an upper bound; 64-bit sums as two 32-bit words,
    // native shared atomics)
    uint32_t* clo = sm + NW * (2 * W * 32 + W);
    uint32_t* chi = clo + W * 32;
    uint32_t* ccnt = chi + W * 32;
    if (ws.sum)
        for (uint32_t x = threadIdx.x; x < W * 32; x += blockDim.x) {
            clo[x] = 0;
            chi[x] = 0;
            ccnt[x] = 0;
        }
    for (uint32_t x = lane; x < W * 32; x += 32) {
        fs[x] = kNone;
        cnt[x] = 0;
    }
    for (uint32_t t = lane; t < W; t += 32) bm[t] = 0;  // W <= 64 words
    __syncthreads();
    const uint32_t kstride = (gridDim.x * blockDim.x) >> 5;
    uint32_t k = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    uint64_t an = 0, bn = 0;  // the next sample's CSR range, loaded one iteration ahead
    if (k < F) {
        an = koff[k];
        bn = koff[k + 1];
    }
    for (; k < F; k += kstride) {
        const uint64_t a = an, b = bn;
        if (k + kstride < F) {
            an = koff[k + kstride];
            bn = koff[k + kstride + 1];
        }
        // the sample's size, issued early (used after the rounds)
        const double szv = (ws.sum && b > a) ? __ldg(ws.sizes + k) : 0.0;
        uint32_t sv[R], xv[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
            if ((uint64_t)r * 32 >= b - a) break;  // warp-uniform: only the rounds in use
            const uint64_t i = a + r * 32 + lane;
            xv[r] = kNone;
            if (i < b) {
                sv[r] = __ldcs(csr + i);
                xv[r] = worker_of_entry(soff, nloc, sv[r], uni);
                atomicMin(&fs[xv[r]], sv[r]);
                atomicAdd(&cnt[xv[r]], 1u);
                atomicOr(&bm[xv[r] >> 5], 1u << (xv[r] & 31));
            }
        }
        __syncwarp();
        // bitmap words: lane l holds word l (W <= 32) or words 2l, 2l+1 (W <= 64)
        const bool two = W > 32;
        const uint32_t w0 = two ? (2 * lane < W ? bm[2 * lane] : 0u) : (lane < W ? bm[lane] : 0u);
        const uint32_t w1 = two && 2 * lane + 1 < W ? bm[2 * lane + 1] : 0u;
        uint32_t pre = 0, total;
        if (W == 1) {
            total = __shfl_sync(0xffffffffu, __popc(w0), 0);
        } else {
            const uint32_t c = __popc(w0) + __popc(w1);
            uint32_t inc = c;
            const uint32_t nl = two ? (W + 1) / 2 : W;  // lanes holding words
            for (uint32_t d = 1; d < nl; d <<= 1) {
                const uint32_t o = __shfl_up_sync(0xffffffffu, inc, d);
                if (lane >= d) inc += o;
            }
            pre = inc - c;
            total = __shfl_sync(0xffffffffu, inc, nl - 1);
        }
        if (lane == 0) pair_count[k] = total;
        unsigned long long sz = 0;
        if (ws.sum && b > a) {
            const double v = szv;
            if (!(v >= 0.0 && v < 0x1.0p40)) {
                if (lane == 0) atomicOr(ws.neg, 1u);  // negative, NaN or huge: no all-fit
            } else {
                sz = __double2ull_ru(v * 0x1.0p20);
            }
        }
#pragma unroll
        for (int r = 0; r < R; ++r) {
            if ((uint64_t)r * 32 >= b - a) break;  // warp-uniform: only the rounds in use
            const uint32_t x = xv[r];
            const uint32_t xw = x != kNone ? x >> 5 : 0u;
            const uint32_t src = two ? xw >> 1 : xw;
            const uint32_t a0 = __shfl_sync(0xffffffffu, w0, W == 1 ? 0u : src);
            const uint32_t a1 = __shfl_sync(0xffffffffu, w1, src);
            const uint32_t pl = W == 1 ? 0u : __shfl_sync(0xffffffffu, pre, src);
            const bool hi = two && (xw & 1u);
            const uint32_t ww = hi ? a1 : a0;
            const uint32_t pw = pl + (hi ? __popc(a0) : 0u);
            if (x != kNone) {
                uint16_t ci = 0, rk = 0xFFFFu;
                if (fs[x] == sv[r]) {
                    ci = (uint16_t)cnt[x];
                    rk = (uint16_t)(pw + __popc(ww & ((1u << (x & 31)) - 1u)));
                    if (ws.sum) {
                        add64(clo + x, chi + x, sz);
                        atomicAdd(&ccnt[x], 1u);
                    }
                }
                const uint64_t i = a + r * 32 + lane;
                einfo[i] = ci;  // CSR order: coalesced (cpos maps stream index -> slot)
                erank[i] = rk;
            }
        }
        __syncwarp();
#pragma unroll
        for (int r = 0; r < R; ++r) {
            if ((uint64_t)r * 32 >= b - a) break;  // warp-uniform: only the rounds in use
            if (xv[r] != kNone) {
                fs[xv[r]] = kNone;
                cnt[xv[r]] = 0;
            }
        }
        for (uint32_t t = lane; t < W; t += 32) bm[t] = 0;  // W <= 64 words
        __syncwarp();
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

// thread per CSR entry: holder records {worker, class, position} at pair_off[k] + rank for the
// pairs' first accesses (k = the stream entry itself).  NP as holder_tile (-1: all-fit uint2).
template <int NP>
__global__ void __launch_bounds__(kThreads) holder_sparse_kernel(
    Part part, uint64_t n, const uint64_t* __restrict__ soff, const uint32_t* __restrict__ stream,
    const uint32_t* __restrict__ csr, const uint16_t* __restrict__ erank, uint32_t MB,
    const uint32_t* __restrict__ rec, uint32_t np_rt, uint32_t J, uint32_t Rp,
    const uint32_t* __restrict__ cbase, const uint64_t* __restrict__ pair_off,
    uint32_t* __restrict__ holders, FastDiv uni, const uint32_t* __restrict__ gate) {
    if (gate && *gate == 0) return;  // speculative all-fit launch, the test failed
    const uint32_t nloc = part.wend - part.wbegin;
    const uint32_t np = NP > 0 ? (uint32_t)NP : np_rt;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t rk = erank[i];
        if (rk == 0xFFFFu) continue;
        const uint32_t s = __ldcs(csr + i);
        const uint32_t k = __ldg(stream + s);
        const uint32_t wl = worker_of_entry(soff, nloc, s, uni);
        const uint32_t w = part.wbegin + wl;
        const uint32_t Le = (uint32_t)part.epoch_len(w);
        const uint32_t rel = (uint32_t)(s - soff[wl]);
        const uint32_t e = rel / Le;
        const uint32_t t = rel - e * Le;
        const uint64_t blk = rec_index(wl, e, nloc, MB, t >> 5);
        const uint32_t bit = t & 31;
        uint32_t cls, pos = 0;
        if constexpr (NP == -1) {
            const uint2 a2 = __ldg(reinterpret_cast<const uint2*>(rec) + blk);
            const uint32_t cb = __ldg(cbase + wl * J);
            cls = (a2.x >> bit) & 1u;
            pos = cls ? a2.y - cb + __popc(a2.x & ((1u << bit) - 1u)) : 0u;
        } else {
            const uint4 v = __ldg(reinterpret_cast<const uint4*>(rec + blk * Rp));
            const uint32_t pl[4] = {v.x, v.y, v.z, v.w};
            cls = 0;
            for (uint32_t q = 0; q < np; ++q) cls |= ((pl[q & 3] >> bit) & 1u) << q;
            uint32_t cm = 0xffffffffu;
            for (uint32_t q = 0; q < np; ++q) cm &= ((cls >> q) & 1u) ? pl[q & 3] : ~pl[q & 3];
            if (cls) {
                const uint32_t wi = np + cls - 1;
                const uint32_t prew = wi < 4 ? pl[wi] : rec[blk * Rp + wi];
                pos = prew - cbase[wl * J + cls - 1] + __popc(cm & ((1u << bit) - 1u));
            }
        }
        uint32_t* h = holders + 3 * (pair_off[k] + rk);
        __stcs(h, w);
        __stcs(h + 1, cls);
        __stcs(h + 2, pos);
    }
}

__global__ void stream_offsets_kernel(Part part, uint64_t* __restrict__ soff) {
    const uint32_t nloc = part.wend - part.wbegin;
    for (uint32_t x = blockIdx.x * blockDim.x + threadIdx.x; x <= nloc; x += gridDim.x * blockDim.x)
        soff[x] = part.stream_offset(part.wbegin + x);
}

// FastDiv by the common per-worker stream length when every local worker has the same one
// (uniform batch slices); d == 1 otherwise (binary search)
static FastDiv uniform_len(const Part& part) {
    const uint64_t L0 = part.epoch_len(part.wbegin), L1 = part.epoch_len(part.wend - 1);
    const uint64_t L = L0 * part.E;
    if (L0 == L1 && L > 1 && L < (1ull << 31) && part.stream_offset(part.wend) < (1ull << 32))
        return FastDiv((uint32_t)L);
    return FastDiv(1u);
}

void launch_sparse_csr(cudaStream_t s, const Part& part, const uint32_t* stream, uint64_t n,
                       uint32_t* cnt, uint64_t* koff, uint32_t* cur, uint32_t* csr, uint32_t* cpos,
                       uint64_t* soff, Workspace& ws) {
    const uint32_t F = part.F, nloc = part.wend - part.wbegin;
    stream_offsets_kernel<<<grid_for(nloc + 1, kThreads), kThreads, 0, s>>>(part, soff);
    cudaMemsetAsync(cnt, 0, (size_t)F * 4, s);
    csr_hist_kernel<<<grid_for(n, kThreads, 148u * 16u), kThreads, 0, s>>>(stream, n, cnt);
    exclusive_scan(s, cnt, F, koff, ws);
    csr_cursor_kernel<<<grid_for(F, kThreads), kThreads, 0, s>>>(koff, F, cur);
    // sample windows of ~64 MB of CSR (samples are uniform over the entries; 64 MB measured
    // best at 115 MB of CSR: 2 windows 1.24 ms, 1 window 1.42, 3 windows 1.29)
    const uint64_t windows = csr_windows(n);
    for (uint64_t j = 0; j < windows; ++j) {
        const uint32_t lo = (uint32_t)(F * j / windows), hi = (uint32_t)(F * (j + 1) / windows);
        csr_scatter_kernel<<<grid_for(n, kThreads, 148u * 16u), kThreads, 0, s>>>(stream, n, lo, hi,
                                                                               cur, csr, cpos);
    }
}

uint64_t csr_windows(uint64_t n) {
    if (const unsigned v = ab_knob("CLAIRPLAN_CSR_WINDOWS", 0)) return std::max(1u, v);  // A/B
    const uint64_t w = std::max<uint64_t>(1, (n * 4 + (64ull << 20) - 1) / (64ull << 20));
    return w <= 16 ? w : 1;  // a CSR of many L2 sizes: one pass (the writes miss L2 anyway)
}

// Sparse passes when they beat the dense E*F ones (B200, config 2 sharded 2/4/8 ways: dense
// ~16 ps per (epoch, sample) cell — inverse rebuild, sample and holder passes; sparse ~55 ps
// per local entry — CSR build, sparse sample and holder passes — growing with the windows).
bool sparse_path_fits(const Part& part) { return (part.wend - part.wbegin) <= 2048 && part.E <= 128; }

bool sparse_path_ok(const Part& part, uint64_t local_entries) {
    if (!sparse_path_fits(part)) return false;
    // the dense inverse / info / rank arrays (8 B per (epoch, sample) cell) would crowd HBM
    if ((double)part.E * (double)part.F * 8.0 > 40e9) return true;
    const uint64_t W = csr_windows(local_entries);
    // (per-window term measured at the ImageNet-22k shape, 128 workers per rank: sparse 29.5 vs
    // dense 26.1 ms with 10 windows; ImageNet-1k, 32 workers: sparse 1.15 vs dense 1.73 ms)
    const double sparse = (double)local_entries * (W == 1 && local_entries * 4 > (64ull << 20) ? 120.0
                                                                                             : 40.0 + 10.0 * (double)W);
    const double dense = 16.0 * (double)part.E * (double)part.F;
    return sparse < dense;
}

void launch_sparse_sample(cudaStream_t s, const Part& part, const uint64_t* soff, const uint64_t* koff,
                          const uint32_t* csr, uint32_t* pair_count, uint16_t* einfo,
                          uint16_t* erank, const WorkerSums& ws) {
    const uint32_t nloc = part.wend - part.wbegin, W = (nloc + 31) / 32;
    const size_t smem = ((size_t)(kThreads / 32) * (2 * W * 32 + W) + 2) * 4 +
                        (ws.sum ? (size_t)W * 32 * 12 : 0);
    // 5 CTAs per SM (48 registers, no spills), two waves (4-way config-2 shard: 1.73 vs
    // 1.84 ms per build with 6 per SM in a 1.33-wave grid)
    static const unsigned gm = ab_knob("CLAIRPLAN_GRID_SPARSE", 10);
    const unsigned grid = grid_for((uint64_t)part.F * 32, kThreads, 148u * gm);
    const FastDiv uni = uniform_len(part);
#define SS_LAUNCH(RV)                                                                              \
    do {                                                                                           \
        allow_smem(sparse_sample_kernel<RV>, \
                             (int)smem);                                                           \
        sparse_sample_kernel<RV><<<grid, kThreads, smem, s>>>(part.F, nloc, W, soff, koff, csr,      \
                                                              pair_count, einfo, erank, ws, uni);  \
    } while (0)
    const uint32_t R = (part.E + 31) / 32;  // a sample has at most one entry per epoch
    if (R == 1) SS_LAUNCH(1);
    else if (R == 2) SS_LAUNCH(2);
    else if (R == 3) SS_LAUNCH(3);
    else SS_LAUNCH(4);
#undef SS_LAUNCH
}

void launch_holder_sparse(cudaStream_t s, const Part& part, uint64_t n, const uint64_t* soff,
                          const uint32_t* stream, const uint32_t* csr, const uint16_t* erank,
                          uint32_t MB, const uint32_t* rec, uint32_t np, uint32_t J, uint32_t Rp,
                          const uint32_t* cbase, const uint64_t* pair_off, uint32_t* holders,
                          bool allfit, const uint32_t* gate) {
    const unsigned grid = grid_for(n, kThreads, 148u * 16u);
    const FastDiv uni = uniform_len(part);
    if (allfit)
        holder_sparse_kernel<-1><<<grid, kThreads, 0, s>>>(part, n, soff, stream, csr, erank, MB, rec,
                                                           np, J, Rp, cbase, pair_off, holders, uni, gate);
    else
        holder_sparse_kernel<0><<<grid, kThreads, 0, s>>>(part, n, soff, stream, csr, erank, MB, rec, np,
                                                          J, Rp, cbase, pair_off, holders, uni, gate);
}

}  // namespace clairplan
