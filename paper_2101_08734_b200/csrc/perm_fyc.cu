// K1-K3 for large F: Fisher-Yates resolution with contiguous target-block buckets ("fyc").
//
// Same resolution as perm.cu (rng.cpp:15-24, access.cpp:52-57): with the
// writers of target y sorted, w_1 < ... < w_m,
//   q(y) = smallest writer != y,   succ(w_k) = w_{k+1},   V(x) = V(q(x)) or x,
//   out[i] = V(succ(i)), or j_i for the last writer of its target,   out[0] = V(0).
// The grouping of the F steps by target is done so that every random access stays inside
// one CTA's shared memory:
//   fyc_part   per tile of 8192 steps: draw j_i, histogram the tile by target block in
//              shared memory, reserve each block's run with ONE global atomic (cursor of the
//              block), write the run into the block's contiguous region.  Blocks have
//              variable width, chosen on the host so that every block expects the same
//              number of writers (target y expects H_F - H_y writers: small targets are
//              heavy), and a capacity of mean + 10 sigma (an overflow is detected and the
//              build reruns on the linked-list path).
//   fyc_block  per target block: its writers in shared memory, counting sort by target,
//              per target the writers in ascending order: q[y] (coalesced), succ of every
//              non-last writer and, tagged, the target itself for the last writer
//              (tsucc[w_m] = y | tag: that step's output, no draw recomputed later), and
//              inv[y] = w_m (coalesced: half of the inverse permutation).
//   fyc_emit   per chunk of steps (warp), chains chased from a shared work list: out[i]
//              for every step, the worker-stream slot, the chased values' inv entries.
// Large F (lg F + lg W > 32): bucket entries hold the step only and fyc_block redraws j_i;
// otherwise (step << lgW) | target-in-block.
#include <cmath>
#include <cstdio>
#include <vector>

#include "internal.h"

namespace clairplan {

constexpr uint32_t kFycPT = 512;                 // threads of fyc_part / fyc_block
constexpr uint32_t kFycK = 14;                   // bucket entries per thread in fyc_block
constexpr uint32_t kFycCap = kFycPT * kFycK;     // 7168 writers per block at most
constexpr uint32_t kFycLoad = 6144;              // expected writers per block
constexpr uint32_t kFycW = 8192;                 // targets per block at most
constexpr uint32_t kFycTK = 16;                  // draws per thread in fyc_part
constexpr uint32_t kFycTS = kFycPT * kFycTK;     // steps per fyc_part tile
constexpr uint32_t kFycLgCell = 8;               // target -> block lookup cells of 256
constexpr uint32_t kFycMaxNB = 24576;            // fyc_part histogram in shared memory
constexpr uint32_t kTag = 0x80000000u;           // tsucc: "this step outputs its target"
constexpr uint32_t kOvf = 0x80000000u;           // rej_flag bit: a block region overflowed

// ---- host geometry -----------------------------------------------------------------------
static double harmonic(double n) {
    if (n < 1) return 0;
    if (n < 64) {
        double h = 0;
        for (int k = 1; k <= (int)n; ++k) h += 1.0 / k;
        return h;
    }
    const double n2 = n * n;
    return std::log(n) + 0.57721566490153286 + 1 / (2 * n) - 1 / (12 * n2) + 1 / (120 * n2 * n2);
}

// expected number of steps writing into targets [0, y): E_0 = H_F - 1, E_t = H_F - H_t
static double expected_writers_below(double F, double HF, double y) {
    if (y <= 0) return 0;
    if (y <= 1) return HF - 1;
    // (H_F - 1) + sum_{t=1}^{y-1} (H_F - H_t), with sum_{t=1}^{n} H_t = (n + 1) H_n - n
    const double n = y - 1;
    return (HF - 1) + n * HF - ((n + 1) * harmonic(n) - n);
}

bool fyc_plan(uint32_t F, FycHost& h) {
    if (F < 2 || F >= 0x80000000u) return false;
    h.F = F;
    h.bstart.clear();
    h.cap.clear();
    const double HF = harmonic((double)F);
    uint32_t y0 = 0;
    double L0 = 0;
    while (y0 < F) {
        const uint32_t hi = (uint32_t)std::min<uint64_t>(F, (uint64_t)y0 + kFycW);
        uint32_t lo = y0 + 1, best = y0 + 1;
        uint32_t a = lo, b = hi;
        while (a <= b) {  // largest y1 in (y0, hi] whose block expects <= kFycLoad writers
            const uint32_t mid = a + (b - a) / 2;
            if (expected_writers_below(F, HF, mid) - L0 <= kFycLoad) {
                best = mid;
                a = mid + 1;
            } else {
                b = mid - 1;
            }
        }
        const double L1 = expected_writers_below(F, HF, best);
        const double mu = std::max(0.0, L1 - L0);
        const double c = std::ceil(mu + 10.0 * std::sqrt(mu) + 64.0);
        h.bstart.push_back(y0);
        h.cap.push_back((uint32_t)std::min<double>(kFycCap, c));
        y0 = best;
        L0 = L1;
    }
    h.NB = (uint32_t)h.cap.size();
    h.bstart.push_back(F);
    if (h.NB > kFycMaxNB) return false;
    h.roff.assign(h.NB + 1, 0);
    for (uint32_t b = 0; b < h.NB; ++b) h.roff[b + 1] = h.roff[b] + h.cap[b];
    h.rtotal = h.roff[h.NB];
    const uint32_t ncell = (F >> kFycLgCell) + 1;
    h.cell.assign(ncell, 0);
    uint32_t b = 0;
    for (uint32_t c = 0; c < ncell; ++c) {
        const uint64_t y = (uint64_t)c << kFycLgCell;
        while (b + 1 < h.NB && h.bstart[b + 1] <= y) ++b;
        h.cell[c] = b;
    }
    uint32_t lgF = 0, lgW = 0;
    while ((1ull << lgF) < F) ++lgF;
    uint32_t wmax = 0;
    for (uint32_t x = 0; x < h.NB; ++x) wmax = std::max(wmax, h.bstart[x + 1] - h.bstart[x]);
    while ((1u << lgW) < wmax) ++lgW;
    h.lgW = lgW;
    h.pack = (lgF + lgW <= 32) ? 1 : 0;
    return true;
}

// ---- device helpers ----------------------------------------------------------------------
__device__ __forceinline__ uint32_t fyc_block_of(const FycDev& g, uint32_t y) {
    uint32_t b = __ldg(g.cell + (y >> kFycLgCell));
    while (__ldg(g.bstart + b + 1) <= y) ++b;
    return b;
}

// exact draw with the rejection-table shift
__device__ __noinline__ uint32_t fyc_draw_exact(uint64_t key, uint32_t e, uint32_t F, uint32_t i,
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

__device__ __forceinline__ uint32_t fyc_draw(uint64_t key, uint32_t e, uint32_t F, uint32_t i,
                                             const uint32_t* st, const uint32_t* cu, uint32_t n,
                                             uint32_t* flag) {
    if (n == 0) {  // no recorded rejection: two 32x32 multiplies; the rejection window -> exact
        const uint64_t x = mix64(key + ((((uint64_t)e) << kEpochShift) + (uint64_t)(F - i)) * kGolden);
        const uint32_t b = i + 1;
        const uint64_t a = (uint64_t)(uint32_t)x * b;
        const uint64_t hh = (uint64_t)(uint32_t)(x >> 32) * b + (a >> 32);
        if (!((uint32_t)hh == 0 && (uint32_t)a < b)) return (uint32_t)(hh >> 32);
    }
    return fyc_draw_exact(key, e, F, i, st, cu, n, flag);
}

// ---- fyc_part ----------------------------------------------------------------------------
// PACK: entries carry the target-in-block (needs the draw kept: 8192-step tiles); otherwise
// only the step is written and each thread keeps just (block, rank) per draw: 16384-step
// tiles, half the block-cursor atomics per step.
template <bool PACK>
__global__ void __launch_bounds__(kFycPT) fyc_part_kernel(uint64_t key, uint32_t F, uint32_t e0,
                                                          FycDev g, RejTable rt,
                                                          uint32_t* __restrict__ rej_flag,
                                                          uint32_t* __restrict__ region,
                                                          uint32_t* __restrict__ cursor) {
    extern __shared__ uint32_t hist[];  // [blocks reachable from this tile]
    const uint32_t t = blockIdx.x, slot = blockIdx.y, e = e0 + slot;
    const uint32_t er = e - rt.e_base;
    const uint32_t* st = rt.step + (size_t)er * rt.cap;
    const uint32_t* cu = rt.cum + (size_t)er * rt.cap;
    const uint32_t nrej = rt.count[er];
    constexpr uint32_t TK = PACK ? kFycTK : 2 * kFycTK, TS = TK * kFycPT;
    constexpr uint32_t RB = PACK ? 13 : 14;  // rank bits (rank < TS)
    const uint32_t i_lo = t * TS, i_hi = min(F, i_lo + TS);
    const uint32_t nbt = fyc_block_of(g, i_hi - 1) + 1;  // j <= i < i_hi
    for (uint32_t b = threadIdx.x; b < nbt; b += kFycPT) hist[b] = 0;
    __syncthreads();
    uint32_t jv[PACK ? TK : 1], bk[TK];
#pragma unroll
    for (uint32_t k0 = 0; k0 < TK; k0 += 8) {  // 8 draws in flight, then their lookups
        uint32_t jj[8];
#pragma unroll
        for (uint32_t u = 0; u < 8; ++u) {
            const uint32_t i = i_lo + (k0 + u) * kFycPT + threadIdx.x;
            jj[u] = (i < i_hi && i > 0) ? fyc_draw(key, e, F, i, st, cu, nrej, rej_flag + er) : kNone;
        }
        // block lookups of the 8 draws issued together: cell, then the first boundary test
        uint32_t bb[8], nx[8];
#pragma unroll
        for (uint32_t u = 0; u < 8; ++u) bb[u] = jj[u] != kNone ? __ldg(g.cell + (jj[u] >> kFycLgCell)) : 0u;
#pragma unroll
        for (uint32_t u = 0; u < 8; ++u) nx[u] = __ldg(g.bstart + bb[u] + 1);
#pragma unroll
        for (uint32_t u = 0; u < 8; ++u) {
            if constexpr (PACK) jv[k0 + u] = jj[u];
            bk[k0 + u] = kNone;
            if (jj[u] != kNone) {
                uint32_t b = bb[u];
                for (uint32_t v = nx[u]; v <= jj[u];) v = __ldg(g.bstart + (++b) + 1);
                const uint32_t r = atomicAdd(&hist[b], 1u);
                bk[k0 + u] = (b << RB) | r;
                if constexpr (PACK) jv[k0 + u] = jj[u] - __ldg(g.bstart + b);
            }
        }
    }
    __syncthreads();
    uint32_t* cur = cursor + (size_t)slot * g.NB;
    for (uint32_t b = threadIdx.x; b < nbt; b += kFycPT) {
        const uint32_t c = hist[b];
        if (c) {
            const uint32_t base = atomicAdd(cur + b, c);
            if (base + c > __ldg(g.cap + b)) atomicOr(rej_flag + er, kOvf);
            hist[b] = base;
        }
    }
    __syncthreads();
    uint32_t* reg = region + (size_t)slot * g.rtotal;
#pragma unroll
    for (uint32_t k = 0; k < TK; ++k) {
        if (bk[k] == kNone) continue;
        const uint32_t b = bk[k] >> RB;
        const uint32_t pos = hist[b] + (bk[k] & ((1u << RB) - 1));
        if (pos < __ldg(g.cap + b)) {
            const uint32_t i = i_lo + k * kFycPT + threadIdx.x;
            if constexpr (PACK) reg[__ldg(g.roff + b) + pos] = (i << g.lgW) | jv[k];
            else reg[__ldg(g.roff + b) + pos] = i;
        }
    }
}

// exclusive scan of a[0..n) in place (n <= kFycW + 1): each thread scans a contiguous run of
// ceil(n / threads) entries, then one scan over the run totals (one barrier pair)
__device__ __forceinline__ void fyc_exscan(uint32_t* a, uint32_t n, uint32_t* wsum) {
    const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr uint32_t NW = kFycPT / 32;
    const uint32_t per = (n + kFycPT - 1) / kFycPT;
    const uint32_t lo = min(n, tid * per), hi = min(n, lo + per);
    uint32_t tot = 0;
    for (uint32_t k = lo; k < hi; ++k) tot += a[k];
    uint32_t inc = tot;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const uint32_t o = __shfl_up_sync(0xffffffffu, inc, d);
        if (lane >= (uint32_t)d) inc += o;
    }
    if (lane == 31) wsum[warp] = inc;
    __syncthreads();
    uint32_t run = inc - tot;
#pragma unroll
    for (uint32_t w = 0; w < NW; ++w) run += w < warp ? wsum[w] : 0u;
    for (uint32_t k = lo; k < hi; ++k) {
        const uint32_t v = a[k];
        a[k] = run;
        run += v;
    }
    __syncthreads();
}

// ---- fyc_block ---------------------------------------------------------------------------
template <bool PACK>
__global__ void __launch_bounds__(kFycPT) fyc_block_kernel(uint64_t key, uint32_t F, uint32_t e0,
                                                           FycDev g, RejTable rt,
                                                           const uint32_t* __restrict__ region,
                                                           const uint32_t* __restrict__ cursor,
                                                           uint32_t* __restrict__ tsucc,
                                                           uint32_t* __restrict__ q,
                                                           uint32_t* __restrict__ inv, int check) {
    extern __shared__ uint32_t sm[];
    __shared__ uint32_t wsum[kFycPT / 32];
    const uint32_t b = blockIdx.x, slot = blockIdx.y, e = e0 + slot;
    const uint32_t y0 = __ldg(g.bstart + b), W = __ldg(g.bstart + b + 1) - y0;
    const uint32_t n = min(cursor[(size_t)slot * g.NB + b], __ldg(g.cap + b));
    if (check && threadIdx.x == 0 && cursor[(size_t)slot * g.NB + b] > __ldg(g.cap + b))
        printf("fyc_block: block %u of epoch %u overflows (%u > cap %u)\n", b, e,
               cursor[(size_t)slot * g.NB + b], __ldg(g.cap + b));
    uint32_t* off = sm;               // [W + 1] counts -> offsets
    uint32_t* S = sm + kFycW + 1;     // [n] writers grouped by target
    const uint32_t* reg = region + (size_t)slot * g.rtotal + __ldg(g.roff + b);
    for (uint32_t x = threadIdx.x; x <= W; x += kFycPT) off[x] = 0;
    __syncthreads();
    const uint32_t er = e - rt.e_base;
    const uint32_t* st = rt.step + (size_t)er * rt.cap;
    const uint32_t* cu = rt.cum + (size_t)er * rt.cap;
    const uint32_t nrej = rt.count[er];
    const uint32_t wmask = (1u << g.lgW) - 1;
    uint32_t iv[kFycK], jr[kFycK];
#pragma unroll
    for (uint32_t k = 0; k < kFycK; ++k) {
        const uint32_t x = threadIdx.x + k * kFycPT;
        iv[k] = x < n ? __ldcs(reg + x) : kNone;
    }
#pragma unroll
    for (uint32_t k = 0; k < kFycK; ++k) {
        jr[k] = kNone;
        if (iv[k] == kNone) continue;
        uint32_t jl;
        if constexpr (PACK) {
            jl = iv[k] & wmask;
            iv[k] >>= g.lgW;
        } else {
            jl = fyc_draw(key, e, F, iv[k], st, cu, nrej, nullptr) - y0;
        }
        if (check && (jl >= W || iv[k] >= F)) {
            printf("fyc_block: entry out of range b=%u e=%u i=%u jl=%u W=%u\n", b, e, iv[k], jl, W);
            continue;
        }
        jr[k] = jl | (atomicAdd(&off[jl], 1u) << 16);  // jl < 8192, rank < 7168
    }
    __syncthreads();
    fyc_exscan(off, W + 1, wsum);  // off[W] = n
#pragma unroll
    for (uint32_t k = 0; k < kFycK; ++k)
        if (jr[k] != kNone) S[off[jr[k] & 0xFFFFu] + (jr[k] >> 16)] = iv[k];
    __syncthreads();
    uint32_t* qq = q + (size_t)slot * F;
    uint32_t* ts = tsucc + (size_t)slot * F;
    uint32_t* irow = inv ? inv + (size_t)e * pitch16(F) : nullptr;
    for (uint32_t t = threadIdx.x; t < W; t += kFycPT) {
        const uint32_t y = y0 + t, beg = off[t], end = off[t + 1];
        if (beg == end) {
            qq[y] = kNone;  // no writer: V(y) = y (a chase root; its inv entry is fyc_emit's)
            continue;
        }
        for (uint32_t a = beg + 1; a < end; ++a) {  // insertion sort (lists are short)
            const uint32_t v = S[a];
            uint32_t c = a;
            while (c > beg && S[c - 1] > v) {
                S[c] = S[c - 1];
                --c;
            }
            S[c] = v;
        }
        const uint32_t w1 = S[beg];
        qq[y] = w1 != y ? w1 : (end - beg > 1 ? S[beg + 1] : kNone);
        for (uint32_t a = beg; a + 1 < end; ++a) ts[S[a]] = S[a + 1];
        const uint32_t wm = S[end - 1];
        ts[wm] = y | kTag;  // out[w_m] = y
        if (irow) irow[y] = wm;
    }
}

// ---- fyc_emit ----------------------------------------------------------------------------
constexpr uint32_t kFycEmitL = 16;
constexpr uint32_t kFycChains = 2;  // chase chains in flight per lane (4: 18.8 vs 18.6 ms, config 4)

__global__ void __launch_bounds__(kThreads, 4) fyc_emit_kernel(Part part, uint32_t e0,
                                                               const uint32_t* __restrict__ tsucc,
                                                               const uint32_t* __restrict__ q,
                                                               uint32_t* __restrict__ inv,
                                                               uint32_t* __restrict__ stream,
                                                               uint32_t* __restrict__ perm_out,
                                                               const StreamDst dst, int check,
                                                               uint32_t* __restrict__ err,
                                                               uint32_t* __restrict__ claim, uint32_t ne) {
    constexpr uint32_t CH = kFycEmitL * 32;
    __shared__ uint32_t sbuf[kThreads / 32][CH];
    __shared__ uint16_t slist[kThreads / 32][CH];
    const uint32_t F = part.F;
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t* buf = sbuf[warp];
    uint16_t* lst = slist[warp];
    const uint32_t nchunk = (F + CH - 1) / CH;
    const uint32_t nwarp = gridDim.x * (blockDim.x >> 5);
    // claim != null: (epoch, chunk) pairs claimed in order by each warp from one counter (the
    // warps in flight stay within ~one epoch's q / inv rows); else blockIdx.y = epoch slot and a
    // grid-stride walk over its chunks
    for (uint32_t it = 0;; ++it) {
        uint32_t slot, c;
        if (claim) {
            uint32_t g = 0;
            if (lane == 0) g = atomicAdd(claim, 1u);
            g = __shfl_sync(0xffffffffu, g, 0);
            slot = g / nchunk;
            c = g - slot * nchunk;
            if (slot >= ne) break;
        } else {
            slot = blockIdx.y;
            c = blockIdx.x * (blockDim.x >> 5) + warp + it * nwarp;
            if (c >= nchunk) break;
        }
        const uint32_t e = e0 + slot;
        const uint32_t* sc = tsucc + (size_t)slot * F;
        const uint32_t* qq = q + (size_t)slot * F;
        const uint32_t cb = c * CH;
        uint32_t sv[kFycEmitL];
#pragma unroll
        for (uint32_t t = 0; t < kFycEmitL; ++t) {
            const uint32_t i = cb + t * 32 + lane;
            sv[t] = i < F ? (i ? __ldcs(sc + i) : 0u) : kTag;  // step 0: V(0), chased from 0
        }
        uint32_t np = 0;
#pragma unroll
        for (uint32_t t = 0; t < kFycEmitL; ++t) {
            const bool chase = !(sv[t] & kTag);
            buf[t * 32 + lane] = sv[t] & ~kTag;
            const uint32_t bal = __ballot_sync(0xffffffffu, chase);
            if (chase) lst[np + __popc(bal & lanemask_lt())] = (uint16_t)(t * 32 + lane);
            np += __popc(bal);
        }
        __syncwarp();
        // kFycChains chains in flight per lane, taken from the chunk's work list in order
        uint32_t nj = lane;
        uint32_t idx[kFycChains], cur[kFycChains];
        bool act[kFycChains];
#pragma unroll
        for (uint32_t c2 = 0; c2 < kFycChains; ++c2) {
            act[c2] = nj < np;
            idx[c2] = act[c2] ? lst[nj] : 0u;
            cur[c2] = act[c2] ? buf[idx[c2]] : 0u;
            nj += 32;
        }
        for (;;) {
            bool any = false;
#pragma unroll
            for (uint32_t c2 = 0; c2 < kFycChains; ++c2) any |= act[c2];
            if (!__any_sync(0xffffffffu, any)) break;
            if (check) {
                bool bad = false;
#pragma unroll
                for (uint32_t c2 = 0; c2 < kFycChains; ++c2) bad |= act[c2] && cur[c2] >= F;
                if (bad) {
                    printf("fyc_emit: chase index out of range e=%u chunk=%u F=%u\n", e, c, F);
                    atomicOr(err, 1u);
                    break;
                }
            }
            uint32_t qv[kFycChains];
#pragma unroll
            for (uint32_t c2 = 0; c2 < kFycChains; ++c2) qv[c2] = act[c2] ? qq[cur[c2]] : 0u;
#pragma unroll
            for (uint32_t c2 = 0; c2 < kFycChains; ++c2) {
                if (!act[c2]) continue;
                if (qv[c2] == kNone) {  // chain ends: V = cur; next chain from the list
                    buf[idx[c2]] = cur[c2];
                    act[c2] = nj < np;
                    if (act[c2]) {
                        idx[c2] = lst[nj];
                        cur[c2] = buf[idx[c2]];
                        nj += 32;
                    }
                } else {
                    cur[c2] = qv[c2];
                }
            }
        }
        __syncwarp();
#pragma unroll 4
        for (uint32_t t = 0; t < kFycEmitL; ++t) {
            const uint32_t i = cb + t * 32 + lane;
            if (i >= F) break;
            const uint32_t v = buf[t * 32 + lane];
            if (check && v >= F) {
                printf("fyc_emit: output out of range e=%u i=%u v=%u sv=%x\n", e, i, v, sv[t]);
                atomicOr(err, 2u);
                continue;
            }
            if (perm_out) perm_out[(size_t)slot * F + i] = v;
            if (inv && !(sv[t] & kTag)) inv[(size_t)e * pitch16(F) + v] = i;  // chase roots only
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

// ---- launcher ----------------------------------------------------------------------------
uint32_t fyc_epochs_per_batch(uint32_t F, uint32_t E) {
    static const uint64_t steps = (uint64_t)ab_knob("CLAIRPLAN_FYC_MSTEPS", 256) << 20;  // A/B
    uint64_t eb = steps / F;  // ~256 M steps per launch: launch tails dominate (config 4: 40 M 50.7, 200 M 49.0 ms)
    if (eb < 1) eb = 1;
    if (eb > E) eb = E;
    if (eb > 128) eb = 128;
    return (uint32_t)eb;
}

void launch_fyc(cudaStream_t s, uint64_t key, const Part& part, uint32_t e0, uint32_t ne,
                const FycDev& g, const RejTable& rt, uint32_t* rej_flag, uint32_t* region,
                uint32_t* cursor, uint32_t* tsucc, uint32_t* q, uint32_t* inv, uint32_t* stream,
                uint32_t* perm_out, const StreamDst* dst) {
    const uint32_t F = part.F;
    static const int check = (int)ab_knob("CLAIRPLAN_FYC_CHECK", 0);  // debug bounds checks
    cudaMemsetAsync(cursor, 0, ((size_t)ne * g.NB + 1) * 4, s);  // + fyc_emit's claim counter
    const uint32_t TS = g.pack ? kFycTS : 2 * kFycTS;
    const uint32_t NT = (F + TS - 1) / TS;
    const size_t sm_part = (size_t)4 * (g.NB + 1);
    const size_t sm_block = (size_t)4 * (kFycW + 1 + kFycCap);
    if (g.pack) {
        allow_smem(fyc_part_kernel<true>, (int)sm_part);
        allow_smem(fyc_block_kernel<true>, (int)sm_block);
        fyc_part_kernel<true><<<dim3(NT, ne), kFycPT, sm_part, s>>>(key, F, e0, g, rt, rej_flag, region, cursor);
        fyc_block_kernel<true><<<dim3(g.NB, ne), kFycPT, sm_block, s>>>(key, F, e0, g, rt, region, cursor,
                                                                        tsucc, q, inv, check);
    } else {
        allow_smem(fyc_part_kernel<false>, (int)sm_part);
        allow_smem(fyc_block_kernel<false>, (int)sm_block);
        fyc_part_kernel<false><<<dim3(NT, ne), kFycPT, sm_part, s>>>(key, F, e0, g, rt, rej_flag, region, cursor);
        fyc_block_kernel<false><<<dim3(g.NB, ne), kFycPT, sm_block, s>>>(key, F, e0, g, rt, region, cursor,
                                                                         tsucc, q, inv, check);
    }
    const StreamDst dloc = dst ? *dst : StreamDst{};
    const uint32_t nchunk = (F + kFycEmitL * 32 - 1) / (kFycEmitL * 32);
    static const bool dyn = ab_knob("CLAIRPLAN_DYN", 1) != 0;  // A/B: per-epoch grid-stride walk
    if (dyn) {
        const uint32_t gx = std::max<uint32_t>(1, std::min<uint64_t>(((uint64_t)nchunk * ne + 7) / 8, 148u * 4u));
        fyc_emit_kernel<<<gx, kThreads, 0, s>>>(part, e0, tsucc, q, inv, stream, perm_out, dloc, check,
                                                rej_flag + (e0 - rt.e_base), cursor + (size_t)ne * g.NB, ne);
    } else {
        dim3 gq(std::max<uint32_t>(1, std::min<uint32_t>((nchunk + 7) / 8, 148u * 8u)), ne);
        fyc_emit_kernel<<<gq, kThreads, 0, s>>>(part, e0, tsucc, q, inv, stream, perm_out, dloc, check,
                                                rej_flag + (e0 - rt.e_base), nullptr, ne);
    }
}

}  // namespace clairplan
