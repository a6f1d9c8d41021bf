// Moving-row gather probe (B200): u8 gathers at random positions of row e of an [E][n] table,
// e advancing with the grid-stride index (the epoch-major order of seg_write3), plus a
// coalesced stream read of the same length.  Compare DRAM bytes (ncu) with the 1-row case.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 row_gather_probe.cu -o row_gather_probe
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hsh(uint64_t x) {
    x ^= x >> 33; x *= 0xff51afd7ed558ccdULL; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ULL; x ^= x >> 33;
    return (uint32_t)x;
}

// MODE 0: grid-stride (index-ordered); MODE 1: CTA-chunked like seg_write3 (each CTA a
// contiguous chunk of `chunk` accesses, chunks taken in order by a resident grid)
template <int MODE>
__global__ void probe(const uint8_t* __restrict__ table, uint64_t n, uint32_t E, const uint32_t* __restrict__ strm,
                      uint32_t* out, uint64_t M, uint64_t chunk) {
    uint32_t acc = 0;
    if (MODE == 0) {
        for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < M; i += (uint64_t)gridDim.x * blockDim.x) {
            const uint32_t e = (uint32_t)((i * E) / M);
            const uint32_t s = strm[i];
            const uint64_t j = ((uint64_t)hsh(i * 0x9E3779B97F4A7C15ULL + s) * n) >> 32;
            acc += table[(uint64_t)e * n + j] + s;
        }
    } else {
        const uint64_t nch = (M + chunk - 1) / chunk;
        for (uint64_t c = blockIdx.x; c < nch; c += gridDim.x) {
            for (uint64_t i = c * chunk + threadIdx.x; i < (c + 1) * chunk && i < M; i += blockDim.x) {
                const uint32_t e = (uint32_t)((i * E) / M);
                const uint32_t s = strm[i];
                const uint64_t j = ((uint64_t)hsh(i * 0x9E3779B97F4A7C15ULL + s) * n) >> 32;
                acc += table[(uint64_t)e * n + j] + s;
            }
        }
    }
    if (acc == 0x12345678u) out[0] = acc;
}

int main(int argc, char** argv) {
    const uint64_t n = (uint64_t)(argc > 1 ? atof(argv[1]) : 14.2) * 1000000;
    const uint32_t E = argc > 2 ? atoi(argv[2]) : 18;
    const int mode = argc > 3 ? atoi(argv[3]) : 0;
    const uint64_t M = (uint64_t)E * n;  // one access per (e, k) like a permutation
    uint8_t* table;
    uint32_t *strm, *out;
    cudaMalloc(&table, (size_t)E * n);
    cudaMalloc(&strm, M * 4);
    cudaMalloc(&out, 4);
    cudaMemset(table, 1, (size_t)E * n);
    cudaMemset(strm, 1, M * 4);
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(a);
        if (mode == 0) probe<0><<<148 * 8, 256>>>(table, n, E, strm, out, M, 0);
        else probe<1><<<148 * 4, 256>>>(table, n, E, strm, out, M, 13900);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (rep == 1) printf("row=%.1f MB E=%u mode=%d  %.3f ms  %.2f G acc/s\n", n / 1e6, E, mode, ms, M / ms / 1e6);
    }
    return 0;
}
