// K1-K3, bucketed resolution (default): the same parallel Fisher-Yates resolution as
// perm.cu (rng.cpp:15-24, access.cpp:52-57), with the grouping of steps by target done in
// shared memory instead of with global atomics and linked-list walks.
//
//   fyb_tile  (per tile of TS steps)  draw j_i, counting-sort the tile's steps by target
//             block (TB targets) in shared memory and write them tile-major:
//             bucket[t*TS + lst[t][b] ...] = (i - t*TS) << lgTB | (j_i mod TB)
//   fyb_block (per target block)      gather the block's runs from every tile, sort by
//             target (shared-memory counting sort; rank/next writer found within the group) and write
//             q[y] = smallest writer != y, succ[w_k] = w_{k+1} (the last writer keeps none:
//             its value is its own draw) and inv[y] = w_m for every target with a writer
//   fyb_emit  (per step)              out[i] = V(succ(i)) (chase through q) or j_i; writes
//             the worker-stream slot, the permutation row and inv of the chase roots (the
//             values no step wrote: V's roots are exactly those).
// Geometry (fy_geometry): TB, TS powers of two with NT*NB cells ~ F/4..F so the runs stay
// a few elements long; valid for F < 2^31 and NB <= kMaxBlocks (else perm.cu's lists path).
#include <cstdlib>

#include "internal.h"

namespace clairplan {

constexpr uint32_t kTileThreads = 512;
constexpr uint32_t kBlockThreads = 256;
constexpr uint32_t kMaxBlocks = 24576;
constexpr uint32_t kMaxTiles = 4096;

bool fy_geometry(uint32_t F, FyGeom& g) {
    if (F < 2 || F >= 0x80000000u) return false;
    uint32_t lgTB = 8;
    while ((1ull << lgTB) * 4096 < F) ++lgTB;
    static const uint32_t max_lgtb = [] {
        const char* v = getenv("CLAIRPLAN_FY_MAXLGTB");  // A/B: bucketed path for larger F
        return v ? (uint32_t)atoi(v) : 11u;
    }();
    if (lgTB > max_lgtb) return false;  // large F: the linked-list path (perm.cu)
    if (const char* v = getenv("CLAIRPLAN_FY_LGTB")) lgTB = (uint32_t)atoi(v);
    const uint64_t TB = 1ull << lgTB;
    uint32_t lgTS = 13;
    while ((1ull << lgTS) * TB < 4ull * F) ++lgTS;
    if (const char* v = getenv("CLAIRPLAN_FY_LGTS")) lgTS = (uint32_t)atoi(v);  // A/B
    if (lgTS + lgTB > 31) return false;
    g.lgTB = lgTB;
    g.lgTS = lgTS;
    g.NB = (uint32_t)((F + TB - 1) >> lgTB);
    g.NT = (uint32_t)((F + (1ull << lgTS) - 1) >> lgTS);
    if (g.NB > kMaxBlocks || g.NT > kMaxTiles) return false;
    // shared-memory capacity of a block's writers (larger blocks use the global pool)
    g.cap = lgTB <= 9 ? 2048 : lgTB == 10 ? 3072 : lgTB == 11 ? 4096 : 8192;
    if (const char* v = getenv("CLAIRPLAN_FY_CAP")) g.cap = (uint32_t)atoi(v);
    return true;
}

// Exclusive scan of a[0..n) in place, T values per round (one per thread, conflict-free);
// all T threads call, returns the total.  wsum: T/32 words.
template <uint32_t T>
__device__ __forceinline__ uint32_t blk_exscan(uint32_t* a, uint32_t n, uint32_t* wsum) {
    const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr uint32_t NW = T / 32;
    uint32_t carry = 0;
    for (uint32_t base = 0; base < n; base += T) {
        const uint32_t k = base + tid;
        const uint32_t v = k < n ? a[k] : 0u;
        uint32_t inc = v;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t o = __shfl_up_sync(0xffffffffu, inc, d);
            if (lane >= (uint32_t)d) inc += o;
        }
        if (lane == 31) wsum[warp] = inc;
        __syncthreads();
        uint32_t wofs = 0, tot = 0;
#pragma unroll
        for (uint32_t w = 0; w < NW; ++w) {
            const uint32_t s = wsum[w];
            wofs += w < warp ? s : 0u;
            tot += s;
        }
        if (k < n) a[k] = carry + wofs + inc - v;
        carry += tot;
        __syncthreads();
    }
    return carry;
}

// Exact draw with the rejection-table shift and the unseen-rejection report (rare path).
__device__ __noinline__ uint32_t fy_draw_exact(uint64_t key, uint32_t e, uint32_t F, uint32_t i,
                                               const uint32_t* st, const uint32_t* cu, uint32_t n,
                                               uint32_t* flag) {
    uint32_t extra;
    const uint32_t j = fy_draw(key, e, F, i, n ? rej_shift(st, cu, n, i) : 0, &extra);
    if (extra && flag) {
        bool known = false;
        for (uint32_t t = 0; t < n; ++t) known |= (st[t] == i);
        if (!known) atomicMax(flag, i + 1);
    }
    return j;
}

struct FyRej {
    const uint32_t* st;
    const uint32_t* cu;
    uint32_t n;
    __device__ __forceinline__ FyRej(const RejTable& rt, uint32_t er)
        : st(rt.step + (size_t)er * rt.cap), cu(rt.cum + (size_t)er * rt.cap), n(rt.count[er]) {}
    // Epochs without recorded rejections (all but ~1e-13 of them): the first draw at position
    // (e << 34) + F - 1 - i, Lemire's product for a 32-bit bound in two 32x32->64 multiplies.
    // Only when the low word of x * (i + 1) is below i + 1 can the draw be a rejection
    // (threshold 2^64 mod (i+1) < i+1, rng.hpp:55-60): that case takes the exact path.
    __device__ __forceinline__ uint32_t draw(uint64_t key, uint32_t e, uint32_t F, uint32_t i,
                                             uint32_t* flag) const {
        if (n == 0) {
            const uint64_t x = mix64(key + ((((uint64_t)e) << kEpochShift) + (uint64_t)(F - i)) * kGolden);
            const uint32_t b = i + 1;
            const uint64_t a = (uint64_t)(uint32_t)x * b;
            const uint64_t h = (uint64_t)(uint32_t)(x >> 32) * b + (a >> 32);
            if (!((uint32_t)h == 0 && (uint32_t)a < b)) return (uint32_t)(h >> 32);
        }
        return fy_draw_exact(key, e, F, i, st, cu, n, flag);
    }
};

// ---- fyb_tile: one tile of TS steps -> tile-major bucket runs --------------------------------
// K > 0: each thread owns K = TS / kTileThreads steps and keeps their draws in registers;
// K == 0: generic tile size, draws recomputed in the second pass.
template <int K>
__global__ void __launch_bounds__(kTileThreads) fyb_tile_kernel(uint64_t key, uint32_t F,
                                                                uint32_t e0, FyGeom g,
                                                                RejTable rt,
                                                                uint32_t* __restrict__ rej_flag,
                                                                uint32_t* __restrict__ bucket,
                                                                uint32_t* __restrict__ lst) {
    extern __shared__ uint32_t sm[];
    __shared__ uint32_t wsum[33];
    const uint32_t t = blockIdx.x, slot = blockIdx.y, e = e0 + slot;
    const uint32_t er = e - rt.e_base;
    const FyRej rj(rt, er);
    const uint32_t TS = 1u << g.lgTS;
    const uint32_t i_lo = t * TS, i_hi = min(F, i_lo + TS);
    const uint32_t nbt = min(g.NB, ((i_hi - 1) >> g.lgTB) + 1);  // j <= i < i_hi
    uint32_t* hist = sm;  // [NB + 1]
    for (uint32_t b = threadIdx.x; b <= nbt; b += kTileThreads) hist[b] = 0;
    __syncthreads();
    const uint32_t tbmask = (1u << g.lgTB) - 1;
    uint32_t jr[K > 0 ? K : 1];
    if constexpr (K > 0) {
#pragma unroll
        for (int k = 0; k < K; ++k) {
            const uint32_t i = i_lo + k * kTileThreads + threadIdx.x;
            jr[k] = (i < i_hi && i > 0) ? rj.draw(key, e, F, i, rej_flag + er) : kNone;
        }
#pragma unroll
        for (int k = 0; k < K; ++k)
            if (jr[k] != kNone) atomicAdd(&hist[jr[k] >> g.lgTB], 1u);
    } else {
        constexpr int U = 8;
        for (uint32_t i0 = i_lo + threadIdx.x; i0 < i_hi; i0 += U * kTileThreads) {
            uint32_t j[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const uint32_t i = i0 + u * kTileThreads;
                j[u] = (i < i_hi && i > 0) ? rj.draw(key, e, F, i, rej_flag + er) : kNone;
            }
#pragma unroll
            for (int u = 0; u < U; ++u)
                if (j[u] != kNone) atomicAdd(&hist[j[u] >> g.lgTB], 1u);
        }
    }
    __syncthreads();
    blk_exscan<kTileThreads>(hist, nbt + 1, wsum);  // hist[nbt] == 0 before: the tile total
    uint32_t* row = lst + ((size_t)slot * g.NT + t) * (g.NB + 1);
    const uint32_t total = hist[nbt];
    for (uint32_t b = threadIdx.x; b <= g.NB; b += kTileThreads) row[b] = b <= nbt ? hist[b] : total;
    __syncthreads();
    if constexpr (K > 0) {  // stage the sorted tile in shared memory, then a coalesced copy-out
        uint32_t* stage = sm + g.NB + 2;
#pragma unroll
        for (int k = 0; k < K; ++k) {
            if (jr[k] == kNone) continue;
            const uint32_t pos = atomicAdd(&hist[jr[k] >> g.lgTB], 1u);
            stage[pos] = ((k * kTileThreads + threadIdx.x) << g.lgTB) | (jr[k] & tbmask);
        }
        __syncthreads();
        uint32_t* out = bucket + (size_t)slot * F + i_lo;
        for (uint32_t k = threadIdx.x; k < total; k += kTileThreads) __stcg(out + k, stage[k]);
    } else {  // scatter straight into the tile's window (L2 merges the sectors)
        uint32_t* out = bucket + (size_t)slot * F + i_lo;
        constexpr int U = 8;
        for (uint32_t i0 = i_lo + threadIdx.x; i0 < i_hi; i0 += U * kTileThreads) {
            uint32_t j[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const uint32_t i = i0 + u * kTileThreads;
                j[u] = (i < i_hi && i > 0) ? rj.draw(key, e, F, i, nullptr) : kNone;
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                if (j[u] == kNone) continue;
                const uint32_t i = i0 + u * kTileThreads;
                const uint32_t pos = atomicAdd(&hist[j[u] >> g.lgTB], 1u);
                out[pos] = ((i - i_lo) << g.lgTB) | (j[u] & tbmask);
            }
        }
    }
}

// ---- fyb_block: one block of TB targets -> q, succ, inv ------------------------------------
// 1. run table: the block's run in every tile t >= tmin (two words of each lst row) and the
//    exclusive scan of the run lengths (element k of the block <-> run r, offset k - rdst[r])
// 2. gather, each warp a contiguous eighth of the elements, 32 at a time (balanced,
//    coalesced: consecutive elements mostly share a run): one binary search per warp finds
//    the first run, the next 32 run starts sit in the lanes and a 5-step shuffle search
//    places every element; each element is pushed on its target's list (head[target], nxt[element]) with
//    a shared atomicExch — no counting sort, no scan
// 3. per writer: walk its target's list for its rank and the next larger writer ->
//    q[y] (smallest writer != y), succ[w] (non-last writers; succ is preset to kNone) and
//    inv[y] = last writer; targets whose list is empty get q = kNone
// BIG: more writers than the shared-memory capacity (blocks of small targets): W/J/nxt live
// in a global pool slab (L2-resident) instead.
template <bool BIG, uint32_t BT>
__device__ __forceinline__ void fyb_block_body(uint32_t F, const FyGeom& g, uint32_t b, uint32_t n,
                                               uint32_t nt, uint32_t tmin, const uint32_t* rsrc,
                                               const uint32_t* rdst, uint32_t* head, uint32_t* W,
                                               uint16_t* J16, uint16_t* N16, uint32_t* J32,
                                               uint32_t* N32, const uint32_t* bk, uint32_t* sc,
                                               uint32_t* qq, uint32_t* iv, bool succ_all) {
    const uint32_t TB = 1u << g.lgTB, tbmask = TB - 1;
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    constexpr uint32_t kEnd = BIG ? kNone : 0xFFFFu;
    // each warp gathers a contiguous range of the block's elements, 32 at a time; one
    // warp-uniform binary search finds the run of its first element, later chunks advance it
    constexpr uint32_t NW = BT / 32;
    const uint32_t xa = (uint32_t)(((uint64_t)n * warp) / NW), xb = (uint32_t)(((uint64_t)n * (warp + 1)) / NW);
    uint32_t r0 = 0;
    if (xa < xb) {
        uint32_t hi = nt;
        while (hi - r0 > 1) {
            const uint32_t mid = (r0 + hi) >> 1;
            if (rdst[mid] <= xa) r0 = mid;
            else hi = mid;
        }
    }
    for (uint32_t x0 = xa; x0 < xb; x0 += 32) {
        while (r0 + 1 < nt && rdst[r0 + 1] <= x0) ++r0;  // warp-uniform, usually 0-1 steps
        const uint32_t r = r0 + lane;
        const uint32_t beg = r < nt ? rdst[r] : n;
        const uint32_t src = r < nt ? rsrc[r] : 0u;
        const uint32_t lim = r0 + 32 < nt ? rdst[r0 + 32] : n;  // runs r0..r0+31 end here
        const uint32_t k = x0 + lane;
        uint32_t j = 0;
#pragma unroll
        for (uint32_t step = 16; step; step >>= 1) {
            const uint32_t bc = __shfl_sync(0xffffffffu, beg, j + step);
            if (bc <= k) j += step;
        }
        uint32_t bj = __shfl_sync(0xffffffffu, beg, j);
        uint32_t sj = __shfl_sync(0xffffffffu, src, j);
        uint32_t rr = r0 + j;
        if (k < xb) {
            if (k >= lim) {  // beyond 32 runs (many empty runs): full search
                uint32_t l2 = r0, h2 = nt;
                while (h2 - l2 > 1) {
                    const uint32_t mid = (l2 + h2) >> 1;
                    if (rdst[mid] <= k) l2 = mid;
                    else h2 = mid;
                }
                rr = l2;
                bj = rdst[rr];
                sj = rsrc[rr];
            }
            const uint32_t v = __ldcs(bk + sj + (k - bj));
            const uint32_t jl = v & tbmask;
            W[k] = ((tmin + rr) << g.lgTS) + (v >> g.lgTB);
            const uint32_t old = atomicExch(&head[jl], k);
            if constexpr (BIG) {
                J32[k] = jl;
                N32[k] = old;
            } else {
                J16[k] = (uint16_t)jl;
                N16[k] = (uint16_t)old;
            }
        }
        r0 = __shfl_sync(0xffffffffu, rr, 31);  // run of the chunk's last element
    }
    __syncthreads();
    const uint32_t y0 = b << g.lgTB;
    for (uint32_t tt = threadIdx.x; tt < TB; tt += BT) {
        const uint32_t y = y0 + tt;
        if (y >= F) break;
        if (head[tt] == kEnd) qq[y] = kNone;  // no writer
    }
    for (uint32_t k = threadIdx.x; k < n; k += BT) {
        const uint32_t w = W[k];
        const uint32_t jl = BIG ? J32[k] : (uint32_t)J16[k];
        bool first = true;
        uint32_t nx = kNone;
        for (uint32_t a = head[jl]; a != kEnd; a = BIG ? N32[a] : (uint32_t)N16[a]) {
            const uint32_t v = W[a];
            first &= !(v < w);
            nx = v > w ? min(nx, v) : nx;
        }
        const uint32_t y = y0 + jl;
        if (first) qq[y] = w != y ? w : nx;   // smallest writer != y
        if (nx == kNone) {
            if (iv) iv[y] = w;                 // the last writer places y (out[w_m] = j = y)
            if (succ_all) sc[w] = kNone;       // every writer's succ written: no preset
        } else {
            sc[w] = nx;
        }
    }
}

template <uint32_t BT>
__global__ void __launch_bounds__(BT) fyb_block_kernel(uint32_t F, FyGeom g,
                                                                  const uint32_t* __restrict__ bucket,
                                                                  const uint32_t* __restrict__ lst,
                                                                  uint32_t* __restrict__ pool,
                                                                  uint32_t* __restrict__ pool_used,
                                                                  uint32_t* __restrict__ succ,
                                                                  uint32_t* __restrict__ q,
                                                                  uint32_t e0,
                                                                  uint32_t* __restrict__ inv,
                                                                  bool succ_all) {
    extern __shared__ uint32_t sm[];
    __shared__ uint32_t wsum[BT / 32];
    __shared__ uint32_t s_pool;
    const uint32_t b = blockIdx.x, slot = blockIdx.y;
    const uint32_t TB = 1u << g.lgTB;
    const uint32_t tmin = (uint32_t)(((uint64_t)b << g.lgTB) >> g.lgTS);
    const uint32_t nt = g.NT - tmin;
    uint32_t* head = sm;                // [TB]
    uint32_t* rdst = head + TB;         // [NT + 1] run offsets within the block
    uint32_t* rsrc = rdst + g.NT + 1;   // [NT] run starts within the epoch's bucket row
    uint32_t* W = rsrc + g.NT;          // [cap]  writer step
    uint16_t* J16 = reinterpret_cast<uint16_t*>(W + g.cap);  // [cap] target within block
    uint16_t* N16 = J16 + g.cap;                              // [cap] next on the target's list
    const uint32_t* rows = lst + (size_t)slot * g.NT * (g.NB + 1);
    for (uint32_t k = threadIdx.x; k < nt; k += BT) {
        const uint32_t* r = rows + (size_t)(tmin + k) * (g.NB + 1) + b;
        const uint32_t lo = r[0];
        rsrc[k] = ((tmin + k) << g.lgTS) + lo;
        rdst[k] = r[1] - lo;
    }
    __syncthreads();
    const uint32_t n = blk_exscan<BT>(rdst, nt, wsum);
    const uint32_t* bk = bucket + (size_t)slot * F;
    uint32_t* sc = succ + (size_t)slot * F;
    uint32_t* qq = q + (size_t)slot * F;
    uint32_t* iv = inv ? inv + (size_t)(e0 + slot) * F : nullptr;
    if (n <= g.cap) {
        for (uint32_t k = threadIdx.x; k < TB / 4; k += BT)
            reinterpret_cast<uint4*>(head)[k] = make_uint4(0xFFFFu, 0xFFFFu, 0xFFFFu, 0xFFFFu);
        __syncthreads();
        fyb_block_body<false, BT>(F, g, b, n, nt, tmin, rsrc, rdst, head, W, J16, N16, nullptr,
                              nullptr, bk, sc, qq, iv, succ_all);
    } else {  // heavy block (small targets): global pool slab
        for (uint32_t k = threadIdx.x; k < TB / 4; k += BT)
            reinterpret_cast<uint4*>(head)[k] = make_uint4(kNone, kNone, kNone, kNone);
        if (threadIdx.x == 0) s_pool = atomicAdd(pool_used + slot, 3 * n);
        __syncthreads();
        uint32_t* gW = pool + (size_t)slot * 4 * F + s_pool;
        fyb_block_body<true, BT>(F, g, b, n, nt, tmin, rsrc, rdst, head, gW, nullptr, nullptr,
                             gW + n, gW + 2 * n, bk, sc, qq, iv, succ_all);
    }
}

// ---- fyb_emit: per step, chase and write --------------------------------------------------
template <int U>  // consecutive positions per thread: one slice lookup serves them
__global__ void __launch_bounds__(kThreads) fyb_emit_kernel(uint64_t key, Part part, uint32_t e0,
                                                            RejTable rt,
                                                            const uint32_t* __restrict__ succ,
                                                            const uint32_t* __restrict__ q,
                                                            uint32_t* __restrict__ inv,
                                                            uint32_t* __restrict__ stream,
                                                            uint32_t* __restrict__ perm_out,
                                                            bool inv_all) {
    const uint32_t slot = blockIdx.y, e = e0 + slot, F = part.F;
    const FyRej rj(rt, e - rt.e_base);
    const uint32_t* sc = succ + (size_t)slot * F;
    const uint32_t* qq = q + (size_t)slot * F;
    const uint32_t nthr = gridDim.x * blockDim.x;
    for (uint32_t i0 = (blockIdx.x * blockDim.x + threadIdx.x) * U; i0 < F; i0 += U * nthr) {
        uint32_t cur[U];
        uint32_t live = 0;
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint32_t i = i0 + u;
            cur[u] = kNone;
            if (i < F) {
                const uint32_t s = i ? __ldcs(sc + i) : 0u;
                if (s == kNone) {
                    cur[u] = rj.draw(key, e, F, i, nullptr);  // last writer of its target
                } else {
                    cur[u] = s;
                    live |= 1u << u;
                }
            }
        }
        const uint32_t chased = live;
        while (live) {
#pragma unroll
            for (int u = 0; u < U; ++u) {
                if (!((live >> u) & 1u)) continue;
                const uint32_t nq = qq[cur[u]];
                if (nq == kNone) live &= ~(1u << u);
                else cur[u] = nq;
            }
        }
        if (perm_out) {
#pragma unroll
            for (int u = 0; u < U; ++u)
                if (i0 + u < F) perm_out[(size_t)slot * F + i0 + u] = cur[u];
        }
        if (inv) {
            // inv_all: every value's position is written here (the epoch's inv row is filled
            // while it is L2-resident); otherwise only the chase roots (fyb_block wrote the rest)
#pragma unroll
            for (int u = 0; u < U; ++u)
                if ((inv_all && i0 + u < F) || ((chased >> u) & 1u)) inv[(size_t)e * F + cur[u]] = i0 + u;
        }
        if (stream && i0 < part.P) {
            uint32_t w, left;
            uint64_t spos;
            part.locate_run(i0, e, w, spos, left);
            if (left >= (uint32_t)U && i0 + U <= part.P) {
                if (w >= part.wbegin && w < part.wend) {
                    uint32_t* dst = stream + part.stream_offset(w) + spos;
#pragma unroll
                    for (int u = 0; u < U; ++u) dst[u] = cur[u];
                }
            } else {
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const uint32_t i = i0 + u;
                    if (i >= part.P) break;
                    part.locate(i, e, w, spos);
                    if (w >= part.wbegin && w < part.wend) stream[part.stream_offset(w) + spos] = cur[u];
                }
            }
        }
    }
}

// ---- fyb_emitq: per warp chunk, chase from a work list ---------------------------------
// fyb_emit's warps wait for the longest of their 64 chains on every iteration (q-chase loads
// are dependent L2 round trips; chain lengths have a long tail).  Here a warp takes a chunk of
// kEmitL * 32 steps: all succ loads of the chunk are issued at once, the draws of the last
// writers are computed, the chunk's chains go to a shared work list and every lane runs
// chains from it, two at a time, until the list is empty, then the chunk's values are written
// back: stream and permutation rows coalesced, inv scattered.  Config 2: 1.20 vs 1.27 ms
// (ncu), 5.85 vs 5.92 ms per plan; CLAIRPLAN_EMITQ=0 selects fyb_emit.
constexpr uint32_t kEmitL = 16;

template <int MINB>
__global__ void __launch_bounds__(kThreads, MINB) fyb_emitq_kernel(uint64_t key, Part part, uint32_t e0,
                                                             RejTable rt,
                                                             const uint32_t* __restrict__ succ,
                                                             const uint32_t* __restrict__ q,
                                                             uint32_t* __restrict__ inv,
                                                             uint32_t* __restrict__ stream,
                                                             uint32_t* __restrict__ perm_out,
                                                             bool inv_all, const StreamDst dst) {
    constexpr uint32_t CH = kEmitL * 32;
    __shared__ uint32_t sbuf[kThreads / 32][CH];
    __shared__ uint16_t slist[kThreads / 32][CH];
    const uint32_t slot = blockIdx.y, e = e0 + slot, F = part.F;
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const FyRej rj(rt, e - rt.e_base);
    const uint32_t* sc = succ + (size_t)slot * F;
    const uint32_t* qq = q + (size_t)slot * F;
    uint32_t* buf = sbuf[warp];
    uint16_t* lst = slist[warp];
    const uint32_t nchunk = (F + CH - 1) / CH;
    const uint32_t nwarp = gridDim.x * (blockDim.x >> 5);
    for (uint32_t c = blockIdx.x * (blockDim.x >> 5) + warp; c < nchunk; c += nwarp) {
        const uint32_t cb = c * CH;
        uint32_t sv[kEmitL];
#pragma unroll
        for (uint32_t t = 0; t < kEmitL; ++t) {
            const uint32_t i = cb + t * 32 + lane;
            sv[t] = i < F ? (i ? __ldcs(sc + i) : 0u) : 0u;
        }
        uint32_t np = 0;
#pragma unroll
        for (uint32_t t = 0; t < kEmitL; ++t) {
            const uint32_t i = cb + t * 32 + lane;
            const bool chase = i < F && sv[t] != kNone;
            uint32_t v = sv[t];
            if (i < F && !chase) v = rj.draw(key, e, F, i, nullptr);  // last writer of its target
            buf[t * 32 + lane] = v;
            const uint32_t bal = __ballot_sync(0xffffffffu, chase);
            if (chase) lst[np + __popc(bal & lanemask_lt())] = (uint16_t)(t * 32 + lane);
            np += __popc(bal);
        }
        __syncwarp();
        // two chains in flight per lane; entries lane, lane + 32, ... taken in order
        uint32_t nj = lane;
        uint32_t idx0 = 0, cur0 = 0, idx1 = 0, cur1 = 0;
        bool a0 = nj < np;
        if (a0) {
            idx0 = lst[nj];
            cur0 = buf[idx0];
        }
        nj += 32;
        bool a1 = nj < np;
        if (a1) {
            idx1 = lst[nj];
            cur1 = buf[idx1];
        }
        nj += 32;
        while (__any_sync(0xffffffffu, a0 || a1)) {
            const uint32_t q0 = a0 ? qq[cur0] : 0u;
            const uint32_t q1 = a1 ? qq[cur1] : 0u;
            if (a0) {
                if (q0 == kNone) {
                    buf[idx0] = cur0;
                    a0 = nj < np;
                    if (a0) {
                        idx0 = lst[nj];
                        cur0 = buf[idx0];
                        nj += 32;
                    }
                } else {
                    cur0 = q0;
                }
            }
            if (a1) {
                if (q1 == kNone) {
                    buf[idx1] = cur1;
                    a1 = nj < np;
                    if (a1) {
                        idx1 = lst[nj];
                        cur1 = buf[idx1];
                        nj += 32;
                    }
                } else {
                    cur1 = q1;
                }
            }
        }
        __syncwarp();
#pragma unroll 4
        for (uint32_t t = 0; t < kEmitL; ++t) {
            const uint32_t i = cb + t * 32 + lane;
            if (i >= F) break;
            const uint32_t v = buf[t * 32 + lane];
            if (perm_out) perm_out[(size_t)slot * F + i] = v;
            if (inv && (inv_all || sv[t] != kNone)) inv[(size_t)e * F + v] = i;
            if ((stream || dst.G) && i < part.P) {
                uint32_t w;
                uint64_t spos;
                part.locate(i, e, w, spos);
                if (w >= part.wbegin && w < part.wend) {
                    const uint64_t idx = part.stream_offset(w) + spos;
                    if (dst.G == 0) {
                        stream[idx] = v;
                    } else {  // the owner's receive buffer (peer memory)
                        uint32_t d = 0;
                        while (d + 1 < dst.G && dst.wb[d + 1] <= w) ++d;
                        dst.base[d][(long long)idx + dst.delta[d]] = v;
                    }
                }
            }
        }
        __syncwarp();
    }
}

// ---- launchers --------------------------------------------------------------------------
size_t fyb_block_smem(const FyGeom& g) {
    return (size_t)4 * ((1u << g.lgTB) + 2 * g.NT + 1 + g.cap) + 4 * (size_t)g.cap;
}

template <int K>
void launch_tile(cudaStream_t s, uint64_t key, uint32_t F, uint32_t e0, uint32_t ne,
                 const FyGeom& g, const RejTable& rt, uint32_t* rej_flag, uint32_t* bucket,
                 uint32_t* lst) {
    const size_t sm = (size_t)4 * (g.NB + 2 + (K > 0 ? (1u << g.lgTS) : 0u));
    cudaFuncSetAttribute(fyb_tile_kernel<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    fyb_tile_kernel<K><<<dim3(g.NT, ne), kTileThreads, sm, s>>>(key, F, e0, g, rt, rej_flag,
                                                                 bucket, lst);
}

void launch_fyb(cudaStream_t s, uint64_t key, const Part& part, uint32_t e0, uint32_t ne,
                const FyGeom& g, const RejTable& rt, uint32_t* rej_flag, uint32_t* bucket,
                uint32_t* lst, uint32_t* pool, uint32_t* pool_used, uint32_t* succ, uint32_t* q,
                uint32_t* inv, uint32_t* stream, uint32_t* perm_out, const StreamDst* dst) {
    const uint32_t F = part.F;
    const StreamDst dloc = dst ? *dst : StreamDst{};
    if (g.lgTS == 13) launch_tile<(1 << 13) / kTileThreads>(s, key, F, e0, ne, g, rt, rej_flag, bucket, lst);
    else if (g.lgTS == 14) launch_tile<(1 << 14) / kTileThreads>(s, key, F, e0, ne, g, rt, rej_flag, bucket, lst);
    else launch_tile<0>(s, key, F, e0, ne, g, rt, rej_flag, bucket, lst);
    cudaMemsetAsync(pool_used, 0, ne * sizeof(uint32_t), s);
    static const bool succ_all = [] {
        const char* v = getenv("CLAIRPLAN_SUCC_ALL");  // A/B: every succ entry from fyb_block
        return v && v[0] == '1';
    }();
    if (!succ_all) cudaMemsetAsync(succ, 0xFF, (size_t)ne * F * sizeof(uint32_t), s);
    const size_t sm_block = fyb_block_smem(g);
    // inv written entirely by fyb_emit (each epoch's row is filled while it is L2-resident;
    // measured 3.46 vs 3.64 ms for the config-2 shuffle stage); CLAIRPLAN_INV_ALL=0: fyb_block
    // writes inv of the targets with a writer, fyb_emit the chase roots (A/B)
    static const bool inv_all = [] {
        const char* v = getenv("CLAIRPLAN_INV_ALL");
        return !(v && v[0] == '0');
    }();
    static const int bt = [] {
        const char* v = getenv("CLAIRPLAN_FYB_THREADS");  // A/B
        return v ? atoi(v) : (int)kBlockThreads;
    }();
#define FYB_LAUNCH(BTV)                                                                           \
    do {                                                                                          \
        cudaFuncSetAttribute(fyb_block_kernel<BTV>, cudaFuncAttributeMaxDynamicSharedMemorySize,   \
                             (int)sm_block);                                                      \
        fyb_block_kernel<BTV><<<dim3(g.NB, ne), BTV, sm_block, s>>>(F, g, bucket, lst, pool,       \
                                                                    pool_used, succ, q, e0,        \
                                                                    inv_all ? nullptr : inv,       \
                                                                    succ_all);                     \
    } while (0)
    if (bt == 128) FYB_LAUNCH(128);
    else if (bt == 512) FYB_LAUNCH(512);
    else FYB_LAUNCH(256);
#undef FYB_LAUNCH
    dim3 grid(grid_for(F, kThreads * 4, 148u * 16u), ne);
    static const int u = [] {
        const char* v = getenv("CLAIRPLAN_EMIT_U");  // A/B (2 measured best for config 2)
        return v ? atoi(v) : 2;
    }();
    static const bool emitq = [] {
        const char* v = getenv("CLAIRPLAN_EMITQ");  // A/B: 0 = fyb_emit (per-thread chains)
        return !(v && v[0] == '0');
    }();
    if (emitq || dloc.G) {  // (the peer-memory stream writes exist in fyb_emitq only)
        const uint32_t nchunk = (F + kEmitL * 32 - 1) / (kEmitL * 32);
        dim3 gq(std::max<uint32_t>(1, std::min<uint32_t>((nchunk + 7) / 8, 148u * 8u)), ne);
        static const int minb = [] {
            const char* v = getenv("CLAIRPLAN_EMITQ_MINB");  // A/B (5: 48 registers, spills)
            return v ? atoi(v) : 4;
        }();
        if (minb == 5)
            fyb_emitq_kernel<5><<<gq, kThreads, 0, s>>>(key, part, e0, rt, succ, q, inv, stream, perm_out, inv_all, dloc);
        else
            fyb_emitq_kernel<4><<<gq, kThreads, 0, s>>>(key, part, e0, rt, succ, q, inv, stream, perm_out, inv_all, dloc);
    } else if (u == 8) {
        dim3 g8(grid_for(F, kThreads * 8, 148u * 16u), ne);
        fyb_emit_kernel<8><<<g8, kThreads, 0, s>>>(key, part, e0, rt, succ, q, inv, stream, perm_out, inv_all);
    } else if (u == 2) {
        dim3 g2(grid_for(F, kThreads * 2, 148u * 16u), ne);
        fyb_emit_kernel<2><<<g2, kThreads, 0, s>>>(key, part, e0, rt, succ, q, inv, stream, perm_out, inv_all);
    } else {
        fyb_emit_kernel<4><<<grid, kThreads, 0, s>>>(key, part, e0, rt, succ, q, inv, stream, perm_out, inv_all);
    }
}

}  // namespace clairplan
