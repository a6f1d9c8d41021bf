// Device-wide exclusive prefix sums (u32/u64 -> u64), used for every offset table of the
// plan (pair offsets = holder_offsets, candidate segment offsets, radix/class tables).
// Three-phase reduce-then-scan: 2048 items per 256-thread block, block sums scanned
// recursively, then a block-local scan with the carried-in prefix.
#include "internal.h"

namespace clairplan {

constexpr int kScanItems = 8;
constexpr int kScanTile = kThreads * kScanItems;

template <typename T>
__device__ __forceinline__ uint64_t block_exclusive_scan(uint64_t v, uint64_t* total) {
    __shared__ uint64_t warp_tot[kThreads / 32];
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint64_t incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint64_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if ((int)lane >= o) incl += y;
    }
    if (lane == 31) warp_tot[warp] = incl;
    __syncthreads();
    uint64_t before = 0, all = 0;
#pragma unroll
    for (int w = 0; w < kThreads / 32; ++w) {
        const uint64_t t = warp_tot[w];
        if (w < (int)warp) before += t;
        all += t;
    }
    __syncthreads();
    *total = all;
    return before + incl - v;
}

template <typename T>
__global__ void __launch_bounds__(kThreads) scan_reduce_kernel(const T* __restrict__ in, uint64_t n,
                                                                uint64_t* __restrict__ bsum) {
    const uint64_t base = (uint64_t)blockIdx.x * kScanTile;
    uint64_t s = 0;
#pragma unroll
    for (int t = 0; t < kScanItems; ++t) {
        const uint64_t i = base + (uint64_t)t * kThreads + threadIdx.x;
        if (i < n) s += (uint64_t)in[i];
    }
    uint64_t tot;
    block_exclusive_scan<T>(s, &tot);
    if (threadIdx.x == 0) bsum[blockIdx.x] = tot;
}

template <typename T>
__global__ void __launch_bounds__(kThreads) scan_apply_kernel(const T* __restrict__ in, uint64_t n,
                                                               const uint64_t* __restrict__ bpre,
                                                               uint64_t* __restrict__ out,
                                                               int write_total) {
    const uint64_t base = (uint64_t)blockIdx.x * kScanTile;
    // thread-contiguous items for a sequential per-thread scan
    uint64_t v[kScanItems];
    uint64_t s = 0;
#pragma unroll
    for (int t = 0; t < kScanItems; ++t) {
        const uint64_t i = base + (uint64_t)threadIdx.x * kScanItems + t;
        v[t] = i < n ? (uint64_t)in[i] : 0;
        s += v[t];
    }
    uint64_t tot;
    uint64_t run = block_exclusive_scan<T>(s, &tot) + (bpre ? bpre[blockIdx.x] : 0);
#pragma unroll
    for (int t = 0; t < kScanItems; ++t) {
        const uint64_t i = base + (uint64_t)threadIdx.x * kScanItems + t;
        if (i < n) out[i] = run;
        run += v[t];
    }
    if (write_total && blockIdx.x == gridDim.x - 1 && threadIdx.x == kThreads - 1) out[n] = run;
}

template <typename T>
void exclusive_scan_impl(cudaStream_t s, const T* in, uint64_t n, uint64_t* out, Workspace& ws) {
    if (n == 0) {
        cudaMemsetAsync(out, 0, sizeof(uint64_t), s);
        return;
    }
    const uint64_t nb = (n + kScanTile - 1) / kScanTile;
    if (nb == 1) {
        scan_apply_kernel<T><<<1, kThreads, 0, s>>>(in, n, nullptr, out, 1);
        return;
    }
    uint64_t* bsum = ws.scratch<uint64_t>(nb + 1);
    scan_reduce_kernel<T><<<(unsigned)nb, kThreads, 0, s>>>(in, n, bsum);
    uint64_t* bpre = ws.scratch<uint64_t>(nb + 1);
    exclusive_scan_impl<uint64_t>(s, bsum, nb, bpre, ws);
    scan_apply_kernel<T><<<(unsigned)nb, kThreads, 0, s>>>(in, n, bpre, out, 1);
}

void exclusive_scan(cudaStream_t s, const uint32_t* in, uint64_t n, uint64_t* out, Workspace& ws) {
    const size_t mark = ws.mark();
    exclusive_scan_impl<uint32_t>(s, in, n, out, ws);
    ws.release(mark);
}
void exclusive_scan(cudaStream_t s, const uint64_t* in, uint64_t n, uint64_t* out, Workspace& ws) {
    const size_t mark = ws.mark();
    exclusive_scan_impl<uint64_t>(s, in, n, out, ws);
    ws.release(mark);
}

}  // namespace clairplan
