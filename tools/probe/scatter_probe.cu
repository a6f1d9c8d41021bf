// Row-scatter probe: E rows of F cells, row e written exactly once per cell in a random order
// (a permutation, like class_write's hp rows / the shuffle's inv rows), rows in sequence, with
// an optional coalesced stream read + stream write of the same length alongside.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void mkperm(uint32_t* p, uint32_t F, uint32_t E) {  // p[e][i] = (a*i + b) mod F (a odd, F prime-ish)
    for (uint64_t x = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; x < (uint64_t)F * E; x += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t e = x / F, i = x % F;
        p[x] = (uint32_t)((i * 2654435761ull + e * 40503ull) % F);
    }
}

template <typename T, int EXTRA>
__global__ void scatter_rows(const uint32_t* __restrict__ perm, T* rows, uint32_t F, uint32_t E,
                             const uint32_t* __restrict__ sin, uint32_t* __restrict__ sout) {
    const uint64_t n = (uint64_t)F * E;
    for (uint64_t x = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; x < n; x += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t k = __ldcs(perm + x);
        const uint64_t e = x / F;
        uint32_t v = (uint32_t)x;
        if (EXTRA) v += __ldcs(sin + x);
        rows[e * F + k] = (T)v;
        if (EXTRA) __stcs(sout + x, v);
    }
}

int main() {
    const uint32_t F = 14197122, E = 24;
    uint32_t *perm, *sin, *sout;
    void* rows;
    cudaMalloc(&perm, (size_t)F * E * 4);
    cudaMalloc(&sin, (size_t)F * E * 4);
    cudaMalloc(&sout, (size_t)F * E * 4);
    cudaMalloc(&rows, (size_t)F * E * 4);
    mkperm<<<148 * 8, 256>>>(perm, F, E);
    cudaMemset(sin, 0, (size_t)F * E * 4);
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    for (int grid : {148 * 2, 148 * 8, 148 * 32})
        for (int v = 0; v < 4; ++v) {
            for (int rep = 0; rep < 2; ++rep) {
                cudaEventRecord(a);
                if (v == 0) scatter_rows<uint16_t, 0><<<grid, 256>>>(perm, (uint16_t*)rows, F, E, sin, sout);
                if (v == 1) scatter_rows<uint16_t, 1><<<grid, 256>>>(perm, (uint16_t*)rows, F, E, sin, sout);
                if (v == 2) scatter_rows<uint32_t, 0><<<grid, 256>>>(perm, (uint32_t*)rows, F, E, sin, sout);
                if (v == 3) scatter_rows<uint32_t, 1><<<grid, 256>>>(perm, (uint32_t*)rows, F, E, sin, sout);
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                float ms;
                cudaEventElapsedTime(&ms, a, b);
                if (rep) printf("grid %5d %s extra=%d  %.3f ms  %.1f G/s\n", grid, v < 2 ? "u16" : "u32", v & 1, ms,
                                (double)F * E / ms / 1e6);
            }
        }
    return 0;
}
