// Gather locality probe: 16-B record gathers from a 7 MB working set laid out contiguously or as
// 1024 chunks of 7 KB spread at a 623 KB stride (the per-epoch block records of the
// ImageNet-22k shape), with a coalesced stream read alongside.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hsh(uint64_t x) {
    x ^= x >> 33; x *= 0xff51afd7ed558ccdULL; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ULL; x ^= x >> 33;
    return (uint32_t)x;
}

__global__ void probe(const uint4* __restrict__ rec, uint64_t chunk_recs, uint64_t stride_recs,
                      uint32_t nchunks, const uint32_t* __restrict__ strm, uint32_t* out, uint64_t M) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < M; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t s = __ldcs(strm + i);
        const uint32_t h = hsh(i * 0x9E3779B97F4A7C15ULL + s);
        const uint32_t c = h % nchunks, r = (h / nchunks) % (uint32_t)chunk_recs;
        const uint4 v = __ldg(rec + c * stride_recs + r);
        __stcs(out + i, v.x + v.y + s);
    }
}

int main() {
    const uint64_t M = 1ull << 28;
    const uint32_t nch = 1024;
    const uint64_t chunk = 433;           // records of 16 B per chunk (7 KB)
    uint4* rec;
    uint32_t *strm, *out;
    cudaMalloc(&rec, 700ull << 20);
    cudaMalloc(&strm, M * 4);
    cudaMalloc(&out, M * 4);
    cudaMemset(rec, 1, 700ull << 20);
    cudaMemset(strm, 0, M * 4);
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    for (uint64_t stride : {433ull, 1024ull, 8192ull, 38970ull}) {  // contiguous .. 623 KB
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(a);
            probe<<<148 * 8, 256>>>(rec, chunk, stride, nch, strm, out, M);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (rep) printf("stride %6llu recs (%7.1f KB): %.3f ms  %.1f G gathers/s\n", (unsigned long long)stride,
                            stride * 16 / 1024.0, ms, M / ms / 1e6);
        }
    }
    return 0;
}
