// TMA tile probe: [E][F] u32 / u16 rows pitched to Fp, boxes of [E][32] moved by tma.cuh's
// helpers and read back through tile_u32 / tile_u16 / tile_quad; checked against the source.
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 tma_probe.cu -o tma_probe
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "tma.cuh"
using namespace clairplan;

__global__ void probe(const __grid_constant__ CUtensorMap m32, const __grid_constant__ CUtensorMap m16,
                      uint32_t E, uint32_t F, uint32_t* out32, uint16_t* out16, uint32_t* outq) {
    extern __shared__ __align__(16) uint8_t smraw[];
    __shared__ uint64_t bar;
    uint8_t* t = smraw + ((1024u - (smem_u32(smraw) & 1023u)) & 1023u);
    const uint32_t o16 = (E * 128u + 1023u) & ~1023u;
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        mbar_fence_init();
    }
    __syncthreads();
    const uint32_t k0 = blockIdx.x * 32;
    if (threadIdx.x == 0) {
        mbar_expect_tx(&bar, E * 192u);
        tma_load_2d(t, &m32, (int32_t)k0, 0, &bar);
        tma_load_2d(t + o16, &m16, (int32_t)k0, 0, &bar);
    }
    mbar_wait(&bar, 0);
    const uint32_t* a = reinterpret_cast<const uint32_t*>(t);
    const uint16_t* b = reinterpret_cast<const uint16_t*>(t + o16);
    for (uint32_t i = threadIdx.x; i < E * 32; i += blockDim.x) {
        const uint32_t e = i / 32, s = i % 32;
        if (k0 + s < F) {
            out32[(size_t)e * F + k0 + s] = tile_u32(a, e, s);
            out16[(size_t)e * F + k0 + s] = tile_u16(b, e, s);
            const uint4 v = tile_quad(a, e, s / 4);
            outq[(size_t)e * F + k0 + s] = quad_at(v, s & 3);
        }
    }
}

int main(int argc, char** argv) {
    const uint32_t E = argc > 1 ? atoi(argv[1]) : 90, F = argc > 2 ? atoi(argv[2]) : 1000;
    const uint32_t Fp = (F + 15) & ~15u;
    std::vector<uint32_t> h32((size_t)E * Fp);
    std::vector<uint16_t> h16((size_t)E * Fp);
    for (uint32_t e = 0; e < E; ++e)
        for (uint32_t k = 0; k < Fp; ++k) {
            h32[(size_t)e * Fp + k] = e * 100000u + k;
            h16[(size_t)e * Fp + k] = (uint16_t)(e * 131u + k * 7u);
        }
    uint32_t *d32, *o32, *oq;
    uint16_t *d16, *o16;
    cudaMalloc(&d32, h32.size() * 4);
    cudaMalloc(&d16, h16.size() * 2);
    cudaMalloc(&o32, (size_t)E * F * 4);
    cudaMalloc(&oq, (size_t)E * F * 4);
    cudaMalloc(&o16, (size_t)E * F * 2);
    cudaMemcpy(d32, h32.data(), h32.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(d16, h16.data(), h16.size() * 2, cudaMemcpyHostToDevice);
    CUtensorMap m32, m16;
    if (!encode_tile_map(&m32, d32, 4, F, E, Fp * 4, 32, E) || !encode_tile_map(&m16, d16, 2, F, E, Fp * 2, 32, E)) {
        printf("encode failed\n");
        return 1;
    }
    const size_t smem = 1024 + ((E * 128u + 1023u) & ~1023u) + E * 64u;
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    probe<<<(F + 31) / 32, 256, smem>>>(m32, m16, E, F, o32, o16, oq);
    cudaError_t err = cudaDeviceSynchronize();
    printf("kernel: %s\n", cudaGetErrorString(err));
    if (err != cudaSuccess) return 1;
    std::vector<uint32_t> r32((size_t)E * F), rq((size_t)E * F);
    std::vector<uint16_t> r16((size_t)E * F);
    cudaMemcpy(r32.data(), o32, r32.size() * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(rq.data(), oq, rq.size() * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(r16.data(), o16, r16.size() * 2, cudaMemcpyDeviceToHost);
    size_t bad = 0;
    for (uint32_t e = 0; e < E; ++e)
        for (uint32_t k = 0; k < F; ++k) {
            const bool ok = r32[(size_t)e * F + k] == h32[(size_t)e * Fp + k] &&
                            rq[(size_t)e * F + k] == h32[(size_t)e * Fp + k] &&
                            r16[(size_t)e * F + k] == h16[(size_t)e * Fp + k];
            if (!ok && bad++ < 5)
                printf("mismatch e=%u k=%u: %u %u %u want %u %u\n", e, k, r32[(size_t)e * F + k], rq[(size_t)e * F + k],
                       r16[(size_t)e * F + k], h32[(size_t)e * Fp + k], h16[(size_t)e * Fp + k]);
        }
    printf("E=%u F=%u mismatches=%zu\n", E, F, bad);
    return bad != 0;
}
