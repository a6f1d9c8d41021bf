// Segmented stable LSD radix pass (8-bit digit) over (key, value) pairs.
//
// Used for
//  - the tier order "count desc, first-access asc" (policies.cpp:154-160): candidates are
//    produced per worker in first-access order, so a stable sort on (maxcount - count) is
//    the reference's stable_sort, one digit for E <= 255 (K5);
//  - the per-class prefetch lists (policies.cpp:31-36,162): a stable partition of the
//    first-access-ordered candidates by class digit (K7);
//  - the generic holder CSR of clairplan_assign_from_streams (policies.cpp:124-142).
//
// Segments are independent (one per worker); tiles of kRadixTile elements never straddle a
// segment.  Per pass: tile histograms laid out (segment, digit, tile) -> one global
// exclusive scan gives every (segment, digit, tile) its output base -> stable scatter with
// __match_any_sync ranks inside each 256-element round.
#include "internal.h"

namespace clairplan {

constexpr int kRadixRound = kThreads;

__global__ void tilemap_count_kernel(const uint64_t* __restrict__ seg_len, uint32_t nseg,
                                     uint32_t tile, uint32_t* __restrict__ ntiles) {
    for (uint32_t s = blockIdx.x * blockDim.x + threadIdx.x; s < nseg; s += gridDim.x * blockDim.x)
        ntiles[s] = (uint32_t)((seg_len[s] + tile - 1) / tile);
}

__global__ void tilemap_fill_kernel(const uint64_t* __restrict__ tile_base, uint32_t nseg,
                                    uint32_t* __restrict__ tile_seg, uint64_t max_tiles) {
    const uint64_t total = tile_base[nseg];
    for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < max_tiles;
         t += (uint64_t)gridDim.x * blockDim.x) {
        if (t >= total) {
            tile_seg[t] = kNone;
            continue;
        }
        uint32_t lo = 0, hi = nseg;  // last s with tile_base[s] <= t
        while (hi - lo > 1) {
            const uint32_t mid = (lo + hi) / 2;
            if (tile_base[mid] <= t) lo = mid;
            else hi = mid;
        }
        tile_seg[t] = lo;
    }
}

void build_tilemap(cudaStream_t s, const uint64_t* seg_len, uint32_t nseg, uint64_t total_len,
                   uint32_t tile, TileMap& tm, Workspace& ws) {
    tm.tile = tile;
    tm.nseg = nseg;
    tm.max_tiles = total_len / tile + nseg + 1;
    uint32_t* nt = ws.scratch<uint32_t>(nseg + 1);
    tm.tile_base = ws.scratch<uint64_t>(nseg + 1);
    tm.tile_seg = ws.scratch<uint32_t>(tm.max_tiles);
    tilemap_count_kernel<<<grid_for(nseg, kThreads), kThreads, 0, s>>>(seg_len, nseg, tile, nt);
    exclusive_scan(s, nt, nseg, tm.tile_base, ws);
    tilemap_fill_kernel<<<grid_for(tm.max_tiles, kThreads), kThreads, 0, s>>>(
        tm.tile_base, nseg, tm.tile_seg, tm.max_tiles);
}

struct TileCtx {
    uint32_t seg, t_local, ntiles_seg;
    uint64_t begin, len, table0;
};

__device__ __forceinline__ bool tile_ctx(const TileMap& tm, const uint64_t* seg_begin,
                                         const uint64_t* seg_len, uint64_t t, TileCtx& c) {
    const uint32_t seg = tm.tile_seg[t];
    if (seg == kNone) return false;
    const uint64_t tb = tm.tile_base[seg];
    c.seg = seg;
    c.t_local = (uint32_t)(t - tb);
    c.ntiles_seg = (uint32_t)(tm.tile_base[seg + 1] - tb);
    const uint64_t off = (uint64_t)c.t_local * tm.tile;
    const uint64_t L = seg_len[seg];
    c.begin = seg_begin[seg] + off;
    c.len = L - off < tm.tile ? L - off : tm.tile;
    c.table0 = 256 * tb;
    return true;
}

__global__ void __launch_bounds__(kThreads) radix_hist_kernel(TileMap tm,
                                                               const uint64_t* __restrict__ seg_begin,
                                                               const uint64_t* __restrict__ seg_len,
                                                               const uint32_t* __restrict__ keys,
                                                               uint32_t shift,
                                                               uint32_t* __restrict__ table) {
    __shared__ uint32_t h[256];
    for (uint64_t t = blockIdx.x; t < tm.max_tiles; t += gridDim.x) {
        TileCtx c;
        if (!tile_ctx(tm, seg_begin, seg_len, t, c)) break;
        h[threadIdx.x] = 0;
        __syncthreads();
        for (uint32_t i = threadIdx.x; i < c.len; i += blockDim.x)
            atomicAdd(&h[(keys[c.begin + i] >> shift) & 255u], 1u);
        __syncthreads();
        table[c.table0 + (uint64_t)threadIdx.x * c.ntiles_seg + c.t_local] = h[threadIdx.x];
        __syncthreads();
    }
}

__global__ void __launch_bounds__(kThreads) radix_scatter_kernel(
    TileMap tm, const uint64_t* __restrict__ seg_begin, const uint64_t* __restrict__ seg_len,
    const uint32_t* __restrict__ keys, const uint32_t* __restrict__ vals, uint32_t shift,
    const uint64_t* __restrict__ scanned, uint32_t* __restrict__ okeys,
    uint32_t* __restrict__ ovals, uint32_t* __restrict__ dest) {
    __shared__ uint32_t run[256];
    __shared__ uint32_t wcnt[kThreads / 32][256];
    __shared__ uint64_t base[256];
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (uint32_t d = threadIdx.x; d < 256; d += blockDim.x) {
        run[d] = 0;
        for (int w = 0; w < kThreads / 32; ++w) wcnt[w][d] = 0;
    }
    for (uint64_t t = blockIdx.x; t < tm.max_tiles; t += gridDim.x) {
        TileCtx c;
        if (!tile_ctx(tm, seg_begin, seg_len, t, c)) break;
        {
            const uint32_t d = threadIdx.x;
            // output base of digit d in this tile, relative to the segment start
            base[d] = seg_begin[c.seg] +
                      (scanned[c.table0 + (uint64_t)d * c.ntiles_seg + c.t_local] - scanned[c.table0]);
            run[d] = 0;
        }
        __syncthreads();
        for (uint32_t r0 = 0; r0 < c.len; r0 += kRadixRound) {
            const uint32_t i = r0 + threadIdx.x;
            const bool valid = i < c.len;
            uint32_t key = 0, val = 0, d = 256 + lane;  // invalid lanes: unique fake digits
            if (valid) {
                key = keys[c.begin + i];
                val = vals ? vals[c.begin + i] : (uint32_t)(c.begin + i);
                d = (key >> shift) & 255u;
            }
            const uint32_t m = __match_any_sync(0xffffffffu, d);
            const uint32_t rank = __popc(m & lanemask_lt());
            if (valid && rank == 0) wcnt[warp][d] = __popc(m);
            __syncthreads();
            if (valid) {
                uint32_t below = 0;
                for (uint32_t w = 0; w < warp; ++w) below += wcnt[w][d];
                const uint64_t pos = base[d] + run[d] + below + rank;
                okeys[pos] = key;
                if (ovals) ovals[pos] = val;
                if (dest) dest[c.begin + i] = (uint32_t)pos;
            }
            __syncthreads();
            {
                const uint32_t dd = threadIdx.x;
                uint32_t s = 0;
#pragma unroll
                for (int w = 0; w < kThreads / 32; ++w) {
                    s += wcnt[w][dd];
                    wcnt[w][dd] = 0;
                }
                run[dd] += s;
            }
            __syncthreads();
        }
    }
}

// One stable pass on digit (key >> shift) & 255.  okeys/ovals may alias nothing of the
// inputs.  `scanned_out` (optional) receives the scanned table for region queries.
void radix_pass(cudaStream_t s, const TileMap& tm, const uint64_t* seg_begin,
                const uint64_t* seg_len, const uint32_t* keys, const uint32_t* vals,
                uint32_t shift, uint32_t* okeys, uint32_t* ovals, uint32_t* dest,
                uint64_t** scanned_out, Workspace& ws) {
    const uint64_t table_n = 256 * tm.max_tiles;
    uint32_t* table = ws.scratch<uint32_t>(table_n);
    uint64_t* scanned = ws.scratch<uint64_t>(table_n + 1);
    cudaMemsetAsync(table, 0, table_n * sizeof(uint32_t), s);
    const unsigned grid = grid_for(tm.max_tiles, 1, 148u * 8u);
    radix_hist_kernel<<<grid, kThreads, 0, s>>>(tm, seg_begin, seg_len, keys, shift, table);
    exclusive_scan(s, table, table_n, scanned, ws);
    radix_scatter_kernel<<<grid, kThreads, 0, s>>>(tm, seg_begin, seg_len, keys, vals, shift,
                                                   scanned, okeys, ovals, dest);
    if (scanned_out) *scanned_out = scanned;
}

// Region [start, end) of digit d inside segment seg after a pass (for class lists).
__global__ void radix_regions_kernel(TileMap tm, const uint64_t* __restrict__ seg_begin,
                                     const uint64_t* __restrict__ seg_len,
                                     const uint64_t* __restrict__ scanned, uint32_t ndig,
                                     uint64_t* __restrict__ rstart, uint64_t* __restrict__ rlen) {
    for (uint64_t x = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; x < (uint64_t)tm.nseg * ndig;
         x += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t seg = (uint32_t)(x / ndig), d = (uint32_t)(x % ndig);
        const uint64_t tb = tm.tile_base[seg];
        const uint32_t nt = (uint32_t)(tm.tile_base[seg + 1] - tb);
        if (nt == 0) {
            rstart[x] = seg_begin[seg];
            rlen[x] = 0;
            continue;
        }
        const uint64_t t0 = 256 * tb;
        const uint64_t a = scanned[t0 + (uint64_t)d * nt] - scanned[t0];
        const uint64_t b = (d + 1 < 256) ? scanned[t0 + (uint64_t)(d + 1) * nt] - scanned[t0]
                                         : seg_len[seg];
        rstart[x] = seg_begin[seg] + a;
        rlen[x] = b - a;
    }
}

void radix_regions(cudaStream_t s, const TileMap& tm, const uint64_t* seg_begin,
                   const uint64_t* seg_len, const uint64_t* scanned, uint32_t ndig,
                   uint64_t* rstart, uint64_t* rlen) {
    radix_regions_kernel<<<grid_for((uint64_t)tm.nseg * ndig, kThreads), kThreads, 0, s>>>(
        tm, seg_begin, seg_len, scanned, ndig, rstart, rlen);
}

}  // namespace clairplan
