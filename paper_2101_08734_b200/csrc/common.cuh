// Shared device/host helpers for the clairplan kernels (sm_100a).
#pragma once
#include <atomic>
#include <cstdlib>
#include <cuda_runtime.h>
#include <stdint.h>

namespace clairplan {

constexpr uint32_t kNone = 0xFFFFFFFFu;
constexpr int kThreads = 256;

// ---- counter PRNG (rng.hpp:16-47) ------------------------------------------------------
constexpr uint64_t kGolden = 0x9e3779b97f4a7c15ULL;
constexpr uint64_t kPermTag = 0x7065726dULL;  // rng.hpp:29
constexpr uint64_t kSizeTag = 0x73697a65ULL;  // rng.hpp:30
constexpr int kEpochShift = 34;               // access.cpp:10

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z ^= z >> 30;
    z *= 0xbf58476d1ce4e5b9ULL;
    z ^= z >> 27;
    z *= 0x94d049bb133111ebULL;
    z ^= z >> 31;
    return z;
}

__host__ __device__ __forceinline__ uint64_t derive_key(uint64_t seed, uint64_t tag) {
    return mix64(seed ^ mix64(tag));
}

__host__ __device__ __forceinline__ uint64_t umulhi64(uint64_t a, uint64_t b) {
#ifdef __CUDA_ARCH__
    return __umul64hi(a, b);
#else
    return (uint64_t)(((unsigned __int128)a * b) >> 64);
#endif
}

// CounterRng::bounded (rng.hpp:50-63) evaluated at an explicit stream position: the draw
// uses position pos+1 (pre-increment), rejections consume further positions. Returns the
// value; *extra = number of rejected draws.
__host__ __device__ __forceinline__ uint64_t bounded_at(uint64_t key, uint64_t pos, uint64_t n,
                                                        uint32_t* extra) {
    uint64_t x = mix64(key + (pos + 1) * kGolden);
    uint64_t lo = x * n;
    uint32_t rej = 0;
    if (lo < n) {
        const uint64_t t = (0 - n) % n;
        while (lo < t) {
            ++rej;
            x = mix64(key + (pos + 1 + rej) * kGolden);
            lo = x * n;
        }
    }
    *extra = rej;
    return umulhi64(x, n);
}

// ---- Fisher-Yates step draw with the per-epoch rejection table --------------------------
// Step i (i = F-1 .. 1) of epoch e draws at position (e << 34) + (F - 1 - i) + shift(i)
// (+1 pre-increment inside bounded_at).  shift(i) = extra draws consumed by steps > i,
// recorded in a tiny table of (step, cumulative extra) sorted by step descending.
struct RejTable {
    const uint32_t* step;  // [cap] per epoch
    const uint32_t* cum;
    const uint32_t* count; // per epoch
    uint32_t cap;
    uint32_t e_base;       // tables are indexed by (epoch - e_base)
};

__host__ __device__ __forceinline__ uint32_t rej_shift(const uint32_t* step, const uint32_t* cum,
                                                       uint32_t n, uint32_t i) {
    uint32_t s = 0;
    for (uint32_t t = 0; t < n; ++t) {
        if (step[t] > i) s = cum[t];
        else break;
    }
    return s;
}

__host__ __device__ __forceinline__ uint32_t fy_draw(uint64_t key, uint32_t e, uint32_t F,
                                                     uint32_t i, uint32_t shift,
                                                     uint32_t* extra) {
    const uint64_t pos = ((uint64_t)e << kEpochShift) + (uint64_t)(F - 1 - i) + shift;
    return (uint32_t)bounded_at(key, pos, (uint64_t)i + 1, extra);
}

// ---- fast unsigned division by a runtime constant (32-bit dividends) ---------------------
// Round-up multiply-shift: q = (umulhi(n, m) + n) >> l with l = ceil(log2 d),
// m = floor(2^32 (2^l - d) / d) + 1; exact for every 32-bit n and d >= 1.
struct FastDiv {
    uint32_t d = 1, m = 1, l = 0;
    FastDiv() = default;
    explicit FastDiv(uint32_t dv) : d(dv) {
        l = 0;
        while ((1ull << l) < dv) ++l;
        m = (uint32_t)(((1ull << 32) * ((1ull << l) - dv)) / dv + 1);
    }
    __host__ __device__ __forceinline__ uint32_t div(uint32_t n) const {
#ifdef __CUDA_ARCH__
        const uint32_t t = __umulhi(n, m);
#else
        const uint32_t t = (uint32_t)(((uint64_t)n * m) >> 32);
#endif
        return (uint32_t)(((uint64_t)t + n) >> l);
    }
};

// ---- partition geometry (access.cpp:14-39, config.cpp:37-44) ----------------------------
struct Part {
    uint32_t F, N, B, E;
    uint32_t drop_last;
    uint64_t full, tail, P;          // T = full batches, tail batch size, covered positions
    uint64_t base, extra;            // batch_slice of a full batch
    uint64_t tbase, textra;          // batch_slice of the tail batch
    uint32_t wbegin, wend;           // worker range of this handle
    uint64_t off0;                   // stream_offset(wbegin)
    uint32_t ebase;                  // first epoch held in the stream (epoch-range streams)
    uint32_t pow2, lgB, lgBase;      // B and base powers of two, no remainder, no tail: shifts
    uint32_t Fp;                     // row pitch of the [E][F] u8/u16 arrays (info, rank): F to 16
    FastDiv dB, dFull1, dFull0, dTail1, dTail0;  // B, base+1, base, tbase+1, tbase

    __host__ __device__ uint64_t len(uint32_t w) const { return base + (w < extra ? 1 : 0); }
    __host__ __device__ uint64_t tlen(uint32_t w) const {
        return tail ? tbase + (w < textra ? 1 : 0) : 0;
    }
    __host__ __device__ uint64_t epoch_len(uint32_t w) const { return full * len(w) + tlen(w); }
    // sum_{w' < w} epoch_len(w')
    __host__ __device__ uint64_t prefix_len(uint32_t w) const {
        const uint64_t mw = w < extra ? w : extra;
        uint64_t s = full * ((uint64_t)w * base + mw);
        if (tail) s += (uint64_t)w * tbase + (w < textra ? w : textra);
        return s;
    }
    __host__ __device__ uint64_t stream_offset(uint32_t w) const {
        return (uint64_t)E * prefix_len(w) - off0;
    }
    // perm position p (< P < 2^32) of epoch e -> worker and position within its stream
    __host__ __device__ __forceinline__ void slice_of(uint32_t p, uint32_t& w, uint32_t& h,
                                                      uint32_t& off) const {
        if (pow2) {  // every slice is `base` long: shifts and masks
            h = p >> lgB;
            const uint32_t o = p & (B - 1);
            w = o >> lgBase;
            off = o & ((1u << lgBase) - 1);
            return;
        }
        h = dB.div(p);
        const uint32_t o = p - h * B;
        const bool tl = h >= full;
        const uint32_t x = (uint32_t)(tl ? textra : extra);
        const uint32_t b1 = (uint32_t)(tl ? tbase : base) + 1;
        const uint32_t big = x * b1;
        if (o < big) {
            w = tl ? dTail1.div(o) : dFull1.div(o);
            off = o - w * b1;
        } else {
            const uint32_t o2 = o - big;
            const uint32_t q = tl ? dTail0.div(o2) : dFull0.div(o2);
            w = x + q;
            off = o2 - q * (b1 - 1);
        }
    }
    __host__ __device__ __forceinline__ void locate(uint64_t p, uint32_t e, uint32_t& w,
                                                    uint64_t& spos) const {
        uint32_t h, off;
        slice_of((uint32_t)p, w, h, off);
        spos = (uint64_t)(e - ebase) * epoch_len(w) + (h < full ? (uint64_t)h * len(w) : full * len(w)) + off;
    }
    // locate plus the number of positions p, p+1, ... that stay in the same batch slice
    // (consecutive stream positions of the same worker)
    __host__ __device__ __forceinline__ void locate_run(uint32_t p, uint32_t e, uint32_t& w,
                                                        uint64_t& spos, uint32_t& left) const {
        uint32_t h, off;
        slice_of(p, w, h, off);
        const bool fl = h < full;
        const uint64_t L = fl ? len(w) : tlen(w);
        spos = (uint64_t)(e - ebase) * epoch_len(w) + (fl ? (uint64_t)h * len(w) : full * len(w)) + off;
        left = (uint32_t)(L - off);
    }
    // worker of position p and the position within that worker's epoch segment
    __host__ __device__ __forceinline__ uint32_t within_epoch(uint32_t p, uint32_t& w) const {
        uint32_t h, off;
        slice_of(p, w, h, off);
        return (uint32_t)((h < full ? (uint64_t)h : full) * len(w)) + off;
    }
    __host__ __device__ __forceinline__ uint32_t worker_of(uint64_t p) const {
        uint32_t w, h, off;
        slice_of((uint32_t)p, w, h, off);
        return w;
    }
};

inline Part make_part(uint32_t F, uint32_t N, uint32_t B, uint32_t E, bool drop_last,
                      uint32_t wbegin, uint32_t wend) {
    Part p{};
    p.F = F; p.N = N; p.B = B; p.E = E; p.drop_last = drop_last ? 1 : 0;
    p.full = F / B;
    p.tail = drop_last ? 0 : F % B;
    p.P = p.full * B + p.tail;
    p.base = B / N; p.extra = B % N;
    p.tbase = p.tail / N; p.textra = p.tail % N;
    p.wbegin = wbegin; p.wend = wend;
    p.dB = FastDiv(B);
    p.dFull1 = FastDiv((uint32_t)p.base + 1);
    p.dFull0 = FastDiv(p.base ? (uint32_t)p.base : 1u);
    p.dTail1 = FastDiv((uint32_t)p.tbase + 1);
    p.dTail0 = FastDiv(p.tbase ? (uint32_t)p.tbase : 1u);
    p.off0 = 0;
    p.ebase = 0;
    p.off0 = p.stream_offset(wbegin);
    auto lg = [](uint64_t v) {
        uint32_t l = 0;
        while ((1ull << l) < v) ++l;
        return l;
    };
    p.lgB = lg(B);
    p.lgBase = lg(p.base);
    p.Fp = (F + 15u) & ~15u;
    p.pow2 = (p.extra == 0 && p.tail == 0 && p.base >= 1 && (1ull << p.lgB) == B &&
              (1ull << p.lgBase) == p.base) ? 1u : 0u;
    return p;
}

// Block records (class bit-planes + class prefix counts per 32-entry block of a (worker, epoch)
// segment) are stored EPOCH-major: one epoch's records of all the handle's workers are
// contiguous (7 MB at the ImageNet-22k shape), so the sample-major passes that gather them one
// epoch at a time stay inside a few 2-MB pages (a per-epoch record set spread worker-major over
// 638 MB gathered 4.5x slower: TLB reach, tools/probe/spread_probe.cu).  The scans over blocks
// (class prefix counts) keep the worker-major block order blk = (wl * E + e) * MB + b.
__host__ __device__ __forceinline__ uint64_t rec_index(uint32_t wl, uint32_t e, uint32_t nloc,
                                                       uint32_t MB, uint32_t b) {
    return ((uint64_t)e * nloc + wl) * MB + b;
}

// Row pitch of the [E][F] per-(epoch, sample) arrays (inverse permutations, info, rank, hp):
// F rounded up to 16 samples, so every row starts 64-B aligned and the sample-major passes
// load 32-sample row pieces with 16-B vector loads (tools/probe/tile_probe.cu: 3.67 vs 1.81
// TB/s for the scalar loads of unaligned rows).
__host__ __device__ __forceinline__ uint64_t pitch16(uint32_t F) { return (uint64_t)((F + 15u) & ~15u); }

// Dynamic shared memory opt-in.  The attribute is per (function, device), not per launch:
// handles built concurrently from several host threads must not lower it under each other
// (thread A sets 20 KB, thread B sets 10 KB, A's 20 KB launch fails with "invalid argument"),
// so every caller raises it to the device's opt-in maximum; a launch's occupancy follows the
// bytes it requests, not this limit.
inline int smem_optin_max() {
    static std::atomic<int> cache[64];
    int dev = 0;
    cudaGetDevice(&dev);
    std::atomic<int>& c = cache[dev & 63];
    int v = c.load(std::memory_order_relaxed);
    if (v == 0) {
        if (cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess || v <= 0)
            v = 48 << 10;
        c.store(v, std::memory_order_relaxed);
    }
    return v;
}
// (the limit is the opt-in maximum less the kernel's static shared memory: a larger value is
// rejected with cudaErrorInvalidValue)
template <typename K>
inline cudaError_t allow_smem(K* kernel, int /*bytes: checked at launch*/) {
    cudaFuncAttributes a;
    cudaError_t e = cudaFuncGetAttributes(&a, reinterpret_cast<const void*>(kernel));
    if (e != cudaSuccess) return e;
    return cudaFuncSetAttribute(reinterpret_cast<const void*>(kernel), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                smem_optin_max() - (int)a.sharedSizeBytes);
}

// ---- small device utilities --------------------------------------------------------------
__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31; }
__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// A/B tuning knobs: read from the environment only in debug builds (make AB_KNOBS=1 defines
// CLAIRPLAN_AB_KNOBS); release builds always use the measured defaults.
inline unsigned ab_knob(const char* name, unsigned def) {
#ifdef CLAIRPLAN_AB_KNOBS
    const char* v = getenv(name);
    return v ? (unsigned)atoi(v) : def;
#else
    (void)name;
    return def;
#endif
}
inline bool ab_flag(const char* name) { return ab_knob(name, 0) != 0; }

// Path selections the parity suite forces to cover every pipeline (documented in DESIGN.md
// §2): CLAIRPLAN_NO_ALLFIT, CLAIRPLAN_FORCE_V1, CLAIRPLAN_DENSE, CLAIRPLAN_FY_LISTS.
inline const char* path_switch(const char* name) { return getenv(name); }

// Grid of a grid-stride kernel whose work order matters (epoch-major passes): never more CTAs
// than can be resident at once, so every CTA walks the work in lockstep with the others.
template <typename K>
inline unsigned resident_grid(K kernel, int threads, size_t smem, unsigned per_sm_cap) {
    int dev = 0, nsm = 148, nb = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kernel, threads, smem);
    if (nb < 1) nb = 1;
    if ((unsigned)nb > per_sm_cap) nb = (int)per_sm_cap;
    return (unsigned)(nb * nsm);
}

inline unsigned grid_for(uint64_t n, unsigned per_block, unsigned cap = 148u * 64u) {
    uint64_t g = (n + per_block - 1) / per_block;
    if (g < 1) g = 1;
    if (g > cap) g = cap;
    return (unsigned)g;
}

}  // namespace clairplan
