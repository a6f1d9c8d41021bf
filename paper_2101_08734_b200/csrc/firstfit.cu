// K6: bit-exact first-fit of the tier-ordered candidates into one cache class
// (pack_first_fit, policies.cpp:40-55):
//     for s in order:  if (s <= remaining) { remaining -= s; take; }
// `remaining -= s` is a chain of IEEE double subtractions; rounding makes it order
// dependent, so a plain parallel prefix sum would not reproduce it.  Exact parallel form:
// while remaining r stays inside one binade [2^k, 2^(k+1)) every r is an integer multiple
// R of u = 2^(k-52), and fl(r - s) = (R - d) u with d = round(s/u) under round-half-even of
// the *result*.  d depends on s and on the parity of R only, so each element is a map
// parity -> (decrement, new parity); these maps compose associatively ("monoid").
//   ff_stats   : per 1024-chunk sum / min / max of sizes
//   ff_prefix  : per worker, approximate r at every chunk start (guess of the binade)
//   ff_agg     : per chunk, the composed map in units of the guessed binade, if the chunk
//                provably stays in it and every size <= 2^k (then every size fits)
//   ff_resolve : one warp per worker walks its chunks with the exact r: O(1) per regular
//                chunk (verified: same binade, result >= 2^52+1 units), skip chunks whose
//                minimum exceeds r, otherwise 32-element sub-chunks with the same two fast
//                paths and an exact sequential fallback (binade crossings, spill zone)
//   ff_expand  : flags of the O(1) chunks
#include <math.h>

#include "internal.h"

namespace clairplan {

constexpr uint32_t kChunk = 1024;  // 256 threads x 4
constexpr int kNoBinade = -100000;

struct Mono {
    long long d0, d1;
    uint32_t p0, p1;
};

__device__ __forceinline__ Mono mono_id() { return Mono{0, 0, 0u, 1u}; }

// s / u = m * 2^(es - (k - 52)) with m the 53-bit significand: integer shifts only.
__device__ __forceinline__ Mono mono_elem(double s, int k) {
    const uint64_t bits = (uint64_t)__double_as_longlong(s);
    const int bexp = (int)((bits >> 52) & 0x7FF);
    uint64_t m = bits & ((1ull << 52) - 1);
    int es;
    if (bexp) {
        m |= 1ull << 52;
        es = bexp - 1075;  // s = m * 2^es
    } else {
        es = -1074;        // subnormal
    }
    const int sh = (k - 52) - es;  // t = m >> sh (s <= 2^k guarantees t <= 2^52)
    long long Di;
    bool up = false, tie = false;
    if (sh <= 0) {
        Di = (long long)(m << (-sh));  // exact integer multiple of u
    } else if (sh >= 64) {
        Di = 0;                        // s < u/2^11: rounds away entirely
    } else {
        Di = (long long)(m >> sh);
        const uint64_t rem = m & ((1ull << sh) - 1);
        const uint64_t half = 1ull << (sh - 1);
        up = rem > half;
        tie = rem == half;
    }
    const uint32_t dpar = (uint32_t)(Di & 1);
    Mono r;
    if (tie) {  // the result R - D - 1/2 rounds to the even neighbour
        r.d0 = Di + (0u ^ dpar);
        r.d1 = Di + (1u ^ dpar);
    } else {
        r.d0 = r.d1 = Di + (up ? 1 : 0);
    }
    r.p0 = (uint32_t)((0 ^ r.d0) & 1);
    r.p1 = (uint32_t)((1 ^ r.d1) & 1);
    return r;
}

// a then b
__device__ __forceinline__ Mono mono_compose(const Mono& a, const Mono& b) {
    Mono r;
    r.d0 = a.d0 + (a.p0 ? b.d1 : b.d0);
    r.p0 = a.p0 ? b.p1 : b.p0;
    r.d1 = a.d1 + (a.p1 ? b.d1 : b.d0);
    r.p1 = a.p1 ? b.p1 : b.p0;
    return r;
}

__device__ __forceinline__ Mono shfl_down_mono(const Mono& m, int o) {
    Mono r;
    r.d0 = __shfl_down_sync(0xffffffffu, m.d0, o);
    r.d1 = __shfl_down_sync(0xffffffffu, m.d1, o);
    r.p0 = __shfl_down_sync(0xffffffffu, m.p0, o);
    r.p1 = __shfl_down_sync(0xffffffffu, m.p1, o);
    return r;
}

// ordered reduction; lane 0 holds the composition lane0 ∘ lane1 ∘ ... ∘ lane31
__device__ __forceinline__ Mono warp_compose(Mono m) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const Mono other = shfl_down_mono(m, o);
        if (((threadIdx.x & 31) & (2 * o - 1)) == 0) m = mono_compose(m, other);
    }
    return m;
}

__device__ __forceinline__ int binade(double r) { return ilogb(r); }

__device__ __forceinline__ double warp_min_d(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

struct FFChunks {
    double *sum, *mn, *mx, *r0;
    int* k;
    long long *d0, *d1;
    uint8_t* pbits;
    uint8_t* status;  // 0 none taken, 1 all taken, 2 explicit flags
    uint8_t* segfit;  // per segment: provably everything fits (skip the exact chain)
};

// GATHER: the sizes are gathered here (sz[i] = src[idx[i]], the tier order's sample ids) and
// written for the later passes, instead of by a separate gather pass over the same chunks
template <bool GATHER>
__global__ void __launch_bounds__(kThreads) ff_stats_kernel(TileMap tm,
                                                             const uint64_t* __restrict__ seg_begin,
                                                             const uint64_t* __restrict__ seg_len,
                                                             double* __restrict__ sz,
                                                             const uint32_t* __restrict__ idx,
                                                             const double* __restrict__ src,
                                                             FFChunks ch) {
    __shared__ double ssum[kThreads / 32], smin[kThreads / 32], smax[kThreads / 32];
    for (uint64_t t = blockIdx.x; t < tm.max_tiles; t += gridDim.x) {
        const uint32_t seg = tm.tile_seg[t];
        if (seg == kNone) break;
        const uint64_t off = (t - tm.tile_base[seg]) * (uint64_t)tm.tile;
        const uint64_t L = seg_len[seg];
        const uint64_t n = L - off < tm.tile ? L - off : tm.tile;
        double* p = sz + seg_begin[seg] + off;
        double s = 0, mn = INFINITY, mx = 0;
        for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
            double v;
            if constexpr (GATHER) {
                v = __ldg(src + __ldcs(idx + seg_begin[seg] + off + i));
                p[i] = v;
            } else {
                v = p[i];
            }
            s += v;
            if (v >= 0.0 && v < INFINITY) {
                mn = fmin(mn, v);
                mx = fmax(mx, v);
            } else {  // negative / NaN / inf: no fast path may touch this chunk (see below)
                mn = -INFINITY;
                mx = INFINITY;
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            s += __shfl_xor_sync(0xffffffffu, s, o);
            mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
            mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        }
        if ((threadIdx.x & 31) == 0) {
            ssum[threadIdx.x >> 5] = s;
            smin[threadIdx.x >> 5] = mn;
            smax[threadIdx.x >> 5] = mx;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            s = ssum[0];
            mn = smin[0];
            mx = smax[0];
            for (int i = 1; i < kThreads / 32; ++i) {
                s += ssum[i];
                mn = fmin(mn, smin[i]);
                mx = fmax(mx, smax[i]);
            }
            ch.sum[t] = s;
            ch.mn[t] = mn;
            ch.mx[t] = mx;
        }
        __syncthreads();
    }
}

// one warp per segment: r0[t] = C - (sum of the segment's earlier chunk sums).  When the whole
// segment's sizes sum (with a generous bound on summation and chain rounding) stays below C,
// every prefix fits, so `s <= remaining` holds at every step and everything is taken.
__global__ void ff_prefix_kernel(TileMap tm, const uint64_t* __restrict__ seg_len, double C,
                                 FFChunks ch) {
    const uint32_t lane = threadIdx.x & 31;
    for (uint32_t seg = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; seg < tm.nseg;
         seg += (gridDim.x * blockDim.x) >> 5) {
        const uint64_t tb = tm.tile_base[seg], te = tm.tile_base[seg + 1];
        double carry = 0, mn = INFINITY;
        for (uint64_t t0 = tb; t0 < te; t0 += 32) {
            const uint64_t t = t0 + lane;
            const double v = t < te ? ch.sum[t] : 0.0;
            if (t < te) mn = fmin(mn, ch.mn[t]);
            double incl = v;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const double y = __shfl_up_sync(0xffffffffu, incl, o);
                if ((int)lane >= o) incl += y;
            }
            if (t < te) ch.r0[t] = C - (carry + incl - v);
            carry += __shfl_sync(0xffffffffu, incl, 31);
        }
        mn = warp_min_d(mn);
        if (lane == 0) {
            const double n = (double)seg_len[seg];
            const double tol = (n + 1024.0) * fmax(C, carry) * 0x1.0p-48;
            ch.segfit[seg] = (mn >= 0.0 && C - carry > tol) ? 1 : 0;
        }
    }
}

// warp per chunk: lane l composes elements [32 l, 32 l + 32) in order (contiguous loads, the
// sectors re-read from L1), then one ordered warp reduction -- no block barriers per chunk
__global__ void __launch_bounds__(kThreads) ff_agg_kernel(TileMap tm,
                                                           const uint64_t* __restrict__ seg_begin,
                                                           const uint64_t* __restrict__ seg_len,
                                                           const double* __restrict__ sz, double C,
                                                           FFChunks ch) {
    static_assert(kChunk == 32 * 32, "ff_agg: 32 elements per lane");
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t nwarp = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t t = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; t < tm.max_tiles; t += nwarp) {
        const uint32_t seg = tm.tile_seg[t];
        if (seg == kNone) break;
        if (ch.segfit[seg]) continue;  // warp-uniform: whole segment fits
        const uint64_t off = (t - tm.tile_base[seg]) * (uint64_t)tm.tile;
        const uint64_t L = seg_len[seg];
        const uint64_t n = L - off < tm.tile ? L - off : tm.tile;
        // binade guess with a generous bound on rounding + summation error
        const double tol = C * (double)(off + 2 * tm.tile) * 0x1.0p-48;
        const double r0 = ch.r0[t], r1 = r0 - ch.sum[t];
        int k = kNoBinade;
        if (r1 - tol > 0) {
            const int k1 = binade(r1 - tol);
            if (binade(r0 + tol) == k1 && k1 > -1000 && ldexp(1.0, k1) >= ch.mx[t]) k = k1;
        }
        if (k == kNoBinade) {  // uniform per warp
            if (lane == 0) ch.k[t] = kNoBinade;
            continue;
        }
        const double* p = sz + seg_begin[seg] + off + (uint64_t)lane * 32;
        const uint32_t cnt = n > lane * 32u ? (n - lane * 32u < 32 ? (uint32_t)(n - lane * 32u) : 32u) : 0u;
        Mono m = mono_id();
        if (cnt == 32) {
#pragma unroll 8
            for (uint32_t i = 0; i < 32; ++i) m = mono_compose(m, mono_elem(p[i], k));
        } else {
            for (uint32_t i = 0; i < cnt; ++i) m = mono_compose(m, mono_elem(p[i], k));
        }
        m = warp_compose(m);
        if (lane == 0) {
            ch.k[t] = k;
            ch.d0[t] = m.d0;
            ch.d1[t] = m.d1;
            ch.pbits[t] = (uint8_t)(m.p0 | (m.p1 << 1));
        }
    }
}

__device__ __forceinline__ double warp_min(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// Applies a composed map to r if it provably stays in binade k; returns false otherwise.
__device__ __forceinline__ bool apply_mono(double& r, int k, long long d0, long long d1) {
    if (!(r > 0) || binade(r) != k) return false;
    const long long R = (long long)ldexp(r, 52 - k);
    const long long R2 = R - ((R & 1) ? d1 : d0);
    if (R2 < (1LL << 52) + 1) return false;
    r = ldexp((double)R2, k - 52);
    return true;
}

__global__ void ff_resolve_kernel(TileMap tm, const uint64_t* __restrict__ seg_begin,
                                  const uint64_t* __restrict__ seg_len,
                                  const double* __restrict__ sz, double C, FFChunks ch,
                                  uint8_t* __restrict__ taken,
                                  unsigned long long* __restrict__ taken_count) {
    const uint32_t lane = threadIdx.x & 31;
    for (uint32_t seg = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; seg < tm.nseg;
         seg += (gridDim.x * blockDim.x) >> 5) {
        const uint64_t tb = tm.tile_base[seg], te = tm.tile_base[seg + 1];
        const uint64_t L = seg_len[seg];
        const double* base = sz + seg_begin[seg];
        uint8_t* flags = taken + seg_begin[seg];
        double r = C;
        unsigned long long ntaken = 0;
        if (ch.segfit[seg]) {
            for (uint64_t t = tb + lane; t < te; t += 32) ch.status[t] = 1;
            if (lane == 0 && taken_count && L) atomicAdd(taken_count, (unsigned long long)L);
            continue;
        }
        for (uint64_t t = tb; t < te; ++t) {
            const uint64_t off = (t - tb) * (uint64_t)tm.tile;
            if (r < ch.mn[t]) {
                if (lane == 0) ch.status[t] = 0;
                continue;
            }
            const int k = ch.k[t];
            if (k != kNoBinade && apply_mono(r, k, ch.d0[t], ch.d1[t])) {
                if (lane == 0) ch.status[t] = 1;
                ntaken += L - off < tm.tile ? L - off : tm.tile;
                continue;
            }
            if (lane == 0) ch.status[t] = 2;
            const uint64_t n = L - off < tm.tile ? L - off : tm.tile;
            for (uint64_t s0 = 0; s0 < n; s0 += 32) {
                const uint64_t i = off + s0 + lane;
                const bool valid = s0 + lane < n;
                const double s = valid ? base[i] : 0.0;
                // the monoid and the skip assume finite non-negative sizes; any other value
                // (policies.cpp:47 `s <= remaining` never takes a NaN and always a negative
                // size) sends the sub-chunk through the exact chain
                const bool odd = __any_sync(0xffffffffu, valid && !(s >= 0.0 && s < INFINITY));
                const double smin = warp_min(valid ? s : INFINITY);
                uint8_t flag = 0;
                if (!odd && r < smin) {
                    if (valid) flags[i] = 0;
                    continue;
                }
                const double smax = warp_max(valid ? s : 0.0);
                bool done = false;
                if (!odd && r > 0) {
                    const int kk = binade(r);
                    if (kk > -1000 && ldexp(1.0, kk) >= smax) {
                        Mono m = valid ? mono_elem(s, kk) : mono_id();
                        m = warp_compose(m);
                        const long long d0 = __shfl_sync(0xffffffffu, m.d0, 0);
                        const long long d1 = __shfl_sync(0xffffffffu, m.d1, 0);
                        if (apply_mono(r, kk, d0, d1)) {
                            flag = 1;
                            done = true;
                        }
                    }
                }
                if (!done) {  // exact sequential chain, identical on every lane
                    for (int j = 0; j < 32; ++j) {
                        const double sj = __shfl_sync(0xffffffffu, s, j);
                        if (s0 + j < n && sj <= r) {
                            r = r - sj;
                            if (j == (int)lane) flag = 1;
                        }
                    }
                }
                if (valid) flags[i] = flag;
                ntaken += __popc(__ballot_sync(0xffffffffu, valid && flag));
            }
        }
        if (lane == 0 && taken_count && ntaken) atomicAdd(taken_count, ntaken);
    }
}

__global__ void __launch_bounds__(kThreads) ff_expand_kernel(TileMap tm,
                                                              const uint64_t* __restrict__ seg_begin,
                                                              const uint64_t* __restrict__ seg_len,
                                                              FFChunks ch,
                                                              uint8_t* __restrict__ taken) {
    for (uint64_t t = blockIdx.x; t < tm.max_tiles; t += gridDim.x) {
        const uint32_t seg = tm.tile_seg[t];
        if (seg == kNone) break;
        const uint8_t st = ch.status[t];
        if (st == 2) continue;
        const uint64_t off = (t - tm.tile_base[seg]) * (uint64_t)tm.tile;
        const uint64_t L = seg_len[seg];
        const uint64_t n = L - off < tm.tile ? L - off : tm.tile;
        uint8_t* p = taken + seg_begin[seg] + off;
        for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) p[i] = st;
    }
}

// taken[seg_begin[w] + i] for every element of every segment: first fit into one class of
// capacity C (same capacity for every worker, SystemConfig is shared).
void first_fit_pass(cudaStream_t s, const uint64_t* seg_begin, const uint64_t* seg_len,
                    uint32_t nseg, uint64_t total, const double* sz, double C, uint8_t* taken,
                    Workspace& ws, unsigned long long* taken_count, const uint32_t* gather_idx,
                    const double* gather_src) {
    TileMap tm;
    build_tilemap(s, seg_len, nseg, total, kChunk, tm, ws);
    FFChunks ch;
    const uint64_t m = tm.max_tiles;
    ch.sum = ws.scratch<double>(m);
    ch.mn = ws.scratch<double>(m);
    ch.mx = ws.scratch<double>(m);
    ch.r0 = ws.scratch<double>(m);
    ch.k = ws.scratch<int>(m);
    ch.d0 = ws.scratch<long long>(m);
    ch.d1 = ws.scratch<long long>(m);
    ch.pbits = ws.scratch<uint8_t>(m);
    ch.status = ws.scratch<uint8_t>(m);
    ch.segfit = ws.scratch<uint8_t>(nseg + 1);
    const unsigned g = grid_for(m, 1, 148u * 64u);
    if (gather_idx)
        ff_stats_kernel<true><<<g, kThreads, 0, s>>>(tm, seg_begin, seg_len, const_cast<double*>(sz),
                                                     gather_idx, gather_src, ch);
    else
        ff_stats_kernel<false><<<g, kThreads, 0, s>>>(tm, seg_begin, seg_len, const_cast<double*>(sz),
                                                      nullptr, nullptr, ch);
    ff_prefix_kernel<<<grid_for((uint64_t)nseg * 32, kThreads), kThreads, 0, s>>>(tm, seg_len, C, ch);
    ff_agg_kernel<<<grid_for(m * 32, kThreads, 148u * 64u), kThreads, 0, s>>>(tm, seg_begin, seg_len, sz, C, ch);
    ff_resolve_kernel<<<grid_for((uint64_t)nseg * 32, 128), 128, 0, s>>>(tm, seg_begin, seg_len,
                                                                         sz, C, ch, taken,
                                                                         taken_count);
    ff_expand_kernel<<<g, kThreads, 0, s>>>(tm, seg_begin, seg_len, ch, taken);
}


// ---- rejects of a pass, in order, for the next class (stable compaction) ----------------
__global__ void __launch_bounds__(kThreads) rej_count_kernel(TileMap tm,
                                                              const uint64_t* __restrict__ seg_begin,
                                                              const uint64_t* __restrict__ seg_len,
                                                              const uint8_t* __restrict__ taken,
                                                              uint32_t* __restrict__ cnt) {
    __shared__ uint32_t ws[kThreads / 32];
    for (uint64_t t = blockIdx.x; t < tm.max_tiles; t += gridDim.x) {
        const uint32_t seg = tm.tile_seg[t];
        if (seg == kNone) {
            if (threadIdx.x == 0) cnt[t] = 0;
            continue;
        }
        const uint64_t off = (t - tm.tile_base[seg]) * (uint64_t)tm.tile;
        const uint64_t L = seg_len[seg];
        const uint64_t n = L - off < tm.tile ? L - off : tm.tile;
        const uint8_t* p = taken + seg_begin[seg] + off;
        uint32_t c = 0;
        for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) c += p[i] == 0;
        c = warp_sum(c);
        if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = c;
        __syncthreads();
        if (threadIdx.x == 0) {
            uint32_t s = 0;
            for (int i = 0; i < kThreads / 32; ++i) s += ws[i];
            cnt[t] = s;
        }
        __syncthreads();
    }
}

__global__ void __launch_bounds__(kThreads) rej_write_kernel(
    TileMap tm, const uint64_t* __restrict__ seg_begin, const uint64_t* __restrict__ seg_len,
    const uint8_t* __restrict__ taken, const uint32_t* __restrict__ seq_idx,
    const uint64_t* __restrict__ base, const double* __restrict__ sorted_size,
    uint64_t out0, uint32_t* __restrict__ out_idx, double* __restrict__ out_sz) {
    __shared__ uint32_t ws[kThreads / 32];
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (uint64_t t = blockIdx.x; t < tm.max_tiles; t += gridDim.x) {
        const uint32_t seg = tm.tile_seg[t];
        if (seg == kNone) break;
        const uint64_t off = (t - tm.tile_base[seg]) * (uint64_t)tm.tile;
        const uint64_t L = seg_len[seg];
        const uint64_t n = L - off < tm.tile ? L - off : tm.tile;
        const uint64_t g = seg_begin[seg] + off;
        uint64_t o = out0 + base[t];
        for (uint32_t r0 = 0; r0 < n; r0 += blockDim.x) {
            const uint32_t i = r0 + threadIdx.x;
            const bool rej = i < n && taken[g + i] == 0;
            const uint32_t bal = __ballot_sync(0xffffffffu, rej);
            if (lane == 0) ws[warp] = __popc(bal);
            __syncthreads();
            uint32_t below = 0, tot = 0;
#pragma unroll
            for (int x = 0; x < kThreads / 32; ++x) {
                below += x < (int)warp ? ws[x] : 0;
                tot += ws[x];
            }
            if (rej) {
                const uint64_t pos = o + below + __popc(bal & lanemask_lt());
                const uint32_t si = seq_idx ? seq_idx[g + i] : (uint32_t)(g + i);
                out_idx[pos] = si;
                out_sz[pos] = sorted_size[si];
            }
            o += tot;
            __syncthreads();
        }
    }
}

__global__ void rej_segments_kernel(TileMap tm, const uint64_t* __restrict__ base,
                                    uint64_t out0, uint64_t* __restrict__ nb,
                                    uint64_t* __restrict__ nl) {
    for (uint32_t s = blockIdx.x * blockDim.x + threadIdx.x; s < tm.nseg; s += gridDim.x * blockDim.x) {
        const uint64_t a = base[tm.tile_base[s]], b = base[tm.tile_base[s + 1]];
        nb[s] = out0 + a;
        nl[s] = b - a;
    }
}

// Rejects (taken == 0) of every segment, stable, into [out0, ...) of out_idx / out_sz;
// their sorted indices (seq_idx maps pass positions to tier order; null = identity) and
// sizes.  New segment bounds in nb / nl.
void compact_rejects(cudaStream_t s, const uint64_t* seg_begin, const uint64_t* seg_len,
                     uint32_t nseg, uint64_t total, const uint8_t* taken, const uint32_t* seq_idx,
                     const double* sorted_size, uint64_t out0, uint32_t* out_idx, double* out_sz,
                     uint64_t* nb, uint64_t* nl, Workspace& ws) {
    TileMap tm;
    build_tilemap(s, seg_len, nseg, total, kChunk, tm, ws);
    uint32_t* cnt = ws.scratch<uint32_t>(tm.max_tiles + 1);
    uint64_t* base = ws.scratch<uint64_t>(tm.max_tiles + 1);
    const unsigned g = grid_for(tm.max_tiles, 1, 148u * 64u);
    rej_count_kernel<<<g, kThreads, 0, s>>>(tm, seg_begin, seg_len, taken, cnt);
    exclusive_scan(s, cnt, tm.max_tiles, base, ws);
    rej_write_kernel<<<g, kThreads, 0, s>>>(tm, seg_begin, seg_len, taken, seq_idx, base,
                                            sorted_size, out0, out_idx, out_sz);
    rej_segments_kernel<<<grid_for(nseg, kThreads), kThreads, 0, s>>>(tm, base, out0, nb, nl);
}

}  // namespace clairplan
