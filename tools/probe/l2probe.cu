// L2 residency probe (B200): random 4-B gathers / scatters over tables of 8..160 MB while a
// coalesced stream of the same length passes (evict-first or normal); time per access and
// (under ncu) DRAM bytes.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 l2probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hsh(uint64_t x) {
    x ^= x >> 33; x *= 0xff51afd7ed558ccdULL; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ULL; x ^= x >> 33;
    return (uint32_t)x;
}

template <int MODE>  // 0 gather, 1 scatter
__global__ void probe(uint32_t* table, uint64_t n, const uint32_t* __restrict__ strm, uint32_t* out,
                      uint64_t M, int ef) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < M; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t s = ef ? __ldcs(strm + i) : strm[i];
        const uint64_t j = ((uint64_t)hsh(i * 0x9E3779B97F4A7C15ULL + s) * n) >> 32;
        if (MODE == 0) {
            const uint32_t v = __ldg(table + j);
            if (ef) __stcs(out + i, v + s); else out[i] = v + s;
        } else {
            table[j] = s + (uint32_t)i;
        }
    }
}

int main() {
    const uint64_t M = 1ull << 28;  // 256M accesses
    uint32_t *table, *strm, *out;
    cudaMalloc(&table, 256ull << 20);
    cudaMalloc(&strm, M * 4);
    cudaMalloc(&out, M * 4);
    cudaMemset(table, 0, 256ull << 20);
    cudaMemset(strm, 1, M * 4);
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    const int mbs[] = {4, 8, 16, 24, 32, 48, 64, 80, 96, 112, 128, 160};
    for (int mode = 0; mode < 2; ++mode)
        for (int ef = 0; ef < 2; ++ef)
            for (int mb : mbs) {
                const uint64_t n = ((uint64_t)mb << 20) / 4;
                for (int rep = 0; rep < 2; ++rep) {
                    cudaEventRecord(a);
                    if (mode == 0) probe<0><<<148 * 16, 256>>>(table, n, strm, out, M, ef);
                    else probe<1><<<148 * 16, 256>>>(table, n, strm, out, M, ef);
                    cudaEventRecord(b);
                    cudaEventSynchronize(b);
                    float ms;
                    cudaEventElapsedTime(&ms, a, b);
                    if (rep == 1)
                        printf("%s ef=%d table=%3d MB  %.3f ms  %.2f G acc/s\n", mode ? "scatter" : "gather ", ef,
                               mb, ms, M / ms / 1e6);
                }
            }
    return 0;
}
