// Sample-major tile reads of an [E][F] u32 array (one 128-B row piece per epoch per tile,
// every row in another 2-MB page) vs the same tiles from a blocked [F/K][E][K] layout (all E
// pieces of a tile inside one page): the TLB cost of the sample passes' access pattern.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <bool BLOCKED>
__global__ void tiles(const uint32_t* __restrict__ a, uint32_t F, uint32_t E, uint32_t K,
                      uint32_t* __restrict__ out) {
    __shared__ uint32_t t[128 * 33];
    uint32_t acc = 0;
    for (uint64_t k0 = (uint64_t)blockIdx.x * 32; k0 < F; k0 += (uint64_t)gridDim.x * 32) {
        __syncthreads();
        for (uint32_t idx = threadIdx.x; idx < E * 32; idx += blockDim.x) {
            const uint32_t e = idx >> 5, l = idx & 31;
            const uint64_t k = k0 + l;
            uint64_t addr;
            if (BLOCKED) addr = (k / K) * (uint64_t)E * K + (uint64_t)e * K + (k % K);
            else addr = (uint64_t)e * F + k;
            t[e * 33 + l] = k < F ? __ldcs(a + addr) : 0u;
        }
        __syncthreads();
        for (uint32_t idx = threadIdx.x; idx < E * 32; idx += blockDim.x) acc += t[(idx & 31) * 33 + (idx >> 5) % E];
    }
    if (acc == 0x12345678u) out[0] = acc;
}

// 16-B loads of a row-pitched [E][Fp] array (rows 16-B aligned): 8 threads per 128-B row piece
__global__ void tiles_vec(const uint32_t* __restrict__ a, uint32_t F, uint32_t Fp, uint32_t E,
                          uint32_t* __restrict__ out) {
    __shared__ uint32_t t[128 * 33];
    uint32_t acc = 0;
    for (uint64_t k0 = (uint64_t)blockIdx.x * 32; k0 < F; k0 += (uint64_t)gridDim.x * 32) {
        __syncthreads();
        for (uint32_t idx = threadIdx.x; idx < E * 8; idx += blockDim.x) {
            const uint32_t e = idx >> 3, q = (idx & 7) * 4;
            const uint4 v = __ldcs(reinterpret_cast<const uint4*>(a + (uint64_t)e * Fp + k0 + q));
            t[e * 33 + q] = v.x; t[e * 33 + q + 1] = v.y; t[e * 33 + q + 2] = v.z; t[e * 33 + q + 3] = v.w;
        }
        __syncthreads();
        for (uint32_t idx = threadIdx.x; idx < E * 32; idx += blockDim.x) acc += t[(idx & 31) * 33 + (idx >> 5) % E];
    }
    if (acc == 0x12345678u) out[0] = acc;
}

int main() {
    const uint32_t F = 14197122, E = 90, K = 4096;
    uint32_t *a, *out;
    const uint64_t n = ((uint64_t)(F + K - 1) / K) * K * E;
    cudaMalloc(&a, n * 4);
    cudaMalloc(&out, 4);
    cudaMemset(a, 1, n * 4);
    cudaEvent_t x, y;
    cudaEventCreate(&x); cudaEventCreate(&y);
    for (int blocked = 0; blocked < 2; ++blocked)
        for (int g : {148 * 4, 148 * 16}) {
            for (int rep = 0; rep < 2; ++rep) {
                cudaEventRecord(x);
                if (blocked) tiles<true><<<g, 256>>>(a, F, E, K, out);
                else tiles<false><<<g, 256>>>(a, F, E, K, out);
                cudaEventRecord(y);
                cudaEventSynchronize(y);
                float ms;
                cudaEventElapsedTime(&ms, x, y);
                if (rep) printf("%s grid %5d: %.3f ms  %.0f GB/s\n", blocked ? "blocked [F/K][E][K]" : "rows [E][F]        ",
                                g, ms, (double)F * E * 4 / ms / 1e6);
            }
        }
    const uint32_t Fp = (F + 15) & ~15u;
    for (int g : {148 * 4, 148 * 8, 148 * 16}) {
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(x);
            tiles_vec<<<g, 256>>>(a, F, Fp, E, out);
            cudaEventRecord(y);
            cudaEventSynchronize(y);
            float ms;
            cudaEventElapsedTime(&ms, x, y);
            if (rep) printf("rows [E][Fp] uint4   grid %5d: %.3f ms  %.0f GB/s\n", g, ms, (double)F * E * 4 / ms / 1e6);
        }
    }
    return 0;
}
