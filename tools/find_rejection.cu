// Searches (seed, epoch, F) for epochs whose Fisher-Yates draws hit a Lemire rejection
// (rng.hpp:54-60: lo < (2^64 mod n)), to freeze a rejection known-answer test.
//   find_rejection F seed epoch_begin epoch_count
// Prints one line per epoch with a rejection: epoch, largest rejecting step i, #rejections
// (draw positions assume no earlier rejection in the epoch, so the largest step is exact).
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include "../paper_2101_08734_b200/csrc/common.cuh"

using namespace clairplan;

__global__ void scan_kernel(uint64_t key, uint32_t F, uint32_t e0, uint32_t ne,
                            unsigned int* maxi, unsigned int* cnt) {
    const uint64_t total = (uint64_t)ne * (F - 1);
    for (uint64_t x = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; x < total;
         x += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t slot = (uint32_t)(x / (F - 1));
        const uint32_t i = 1 + (uint32_t)(x % (F - 1));
        const uint32_t e = e0 + slot;
        const uint64_t n = (uint64_t)i + 1;
        const uint64_t pos = ((uint64_t)e << kEpochShift) + (uint64_t)(F - 1 - i) + 1;
        const uint64_t xv = mix64(key + pos * kGolden);
        const uint64_t lo = xv * n;
        if (lo < n) {
            const uint64_t t = (0 - n) % n;
            if (lo < t) {
                atomicMax(&maxi[slot], i);
                atomicAdd(&cnt[slot], 1u);
            }
        }
    }
}

int main(int argc, char** argv) {
    if (argc < 5) {
        std::fprintf(stderr, "usage: %s F seed epoch_begin epoch_count\n", argv[0]);
        return 2;
    }
    const uint32_t F = (uint32_t)strtoul(argv[1], nullptr, 10);
    const uint64_t seed = strtoull(argv[2], nullptr, 10);
    const uint32_t e0 = (uint32_t)strtoul(argv[3], nullptr, 10);
    const uint32_t ne = (uint32_t)strtoul(argv[4], nullptr, 10);
    const uint64_t key = derive_key(seed, kPermTag);
    unsigned int *maxi, *cnt;
    cudaMalloc(&maxi, ne * 4);
    cudaMalloc(&cnt, ne * 4);
    cudaMemset(maxi, 0, ne * 4);
    cudaMemset(cnt, 0, ne * 4);
    scan_kernel<<<148 * 32, 256>>>(key, F, e0, ne, maxi, cnt);
    cudaDeviceSynchronize();
    unsigned int* hm = new unsigned int[ne];
    unsigned int* hc = new unsigned int[ne];
    cudaMemcpy(hm, maxi, ne * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(hc, cnt, ne * 4, cudaMemcpyDeviceToHost);
    int found = 0;
    for (uint32_t s = 0; s < ne; ++s)
        if (hc[s]) {
            std::printf("F=%u seed=%llu epoch=%u max_step=%u rejections=%u\n", F,
                        (unsigned long long)seed, e0 + s, hm[s], hc[s]);
            ++found;
        }
    std::printf("searched %u epochs, %d with rejections\n", ne, found);
    return 0;
}
