// K4a: per-sample pass over the inverse permutations — the (worker, sample) histogram.
//
// For sample k, inv[e][k] is its position in epoch e's permutation, hence (through the
// partition) the worker that reads it in epoch e.  Grouping the <= E accesses of k by worker
// gives, for every distinct (w, k) pair, its access count (access_frequencies,
// access.cpp:80-88) and its first epoch, which is where its first stream position lies
// (first_access_positions, policies.cpp:16-23: positions grow with the epoch).  It also
// gives the pair's rank among k's distinct workers in ascending worker order, which is the
// pair's slot in the holder CSR (build_index, policies.cpp:124-142, worker-major order).
//
// One CTA takes 32 consecutive samples: their E x 32 inverse entries are loaded with
// coalesced 128-B rows into shared memory, one warp processes one sample at a time with
// lanes = epochs (__match_any_sync groups equal workers inside a 32-epoch round, a per-warp
// shared-memory hash keyed by worker merges rounds, a per-warp worker bitmap with prefix
// popcounts gives the ranks), and the tile is written back in place as
//     info[e][k] = (count << 16) | rank   at the pair's first epoch, 0 elsewhere.
// pair_count[k] = number of distinct workers (of this handle's range) reading k.
#include "internal.h"

namespace clairplan {

__device__ __forceinline__ uint32_t hash_slot(uint32_t w, uint32_t mask) {
    return (w * 0x9E3779B1u >> 7) & mask;
}

__global__ void __launch_bounds__(kThreads) sample_pass_kernel(Part part,
                                                                uint32_t* __restrict__ info,
                                                                uint32_t* __restrict__ pair_count,
                                                                uint32_t hs, uint32_t nw_words) {
    extern __shared__ uint32_t smem[];
    const uint32_t E = part.E, F = part.F;
    const uint32_t nwarps = blockDim.x >> 5;
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint32_t* T = smem;                                  // [E][32]
    uint32_t* wbase = T + (size_t)E * 32 + (size_t)warp * (2 * hs + 2 * nw_words);
    uint32_t* keys = wbase;
    uint32_t* vals = keys + hs;
    uint32_t* bm = vals + hs;
    uint32_t* pre = bm + nw_words;
    const uint32_t mask = hs - 1;
    const uint32_t rounds = (E + 31) / 32;

    for (uint32_t t = lane; t < hs; t += 32) keys[t] = kNone;
    for (uint32_t t = lane; t < nw_words; t += 32) bm[t] = 0;

    for (uint64_t k0 = (uint64_t)blockIdx.x * 32; k0 < F; k0 += (uint64_t)gridDim.x * 32) {
        __syncthreads();
        for (uint32_t idx = threadIdx.x; idx < E * 32; idx += blockDim.x) {
            const uint32_t e = idx >> 5, l = idx & 31;
            T[idx] = (k0 + l < F) ? info[(size_t)e * pitch16(F) + k0 + l] : kNone;
        }
        __syncthreads();
        for (uint32_t s = warp; s < 32; s += nwarps) {
            if (k0 + s >= F) break;
            uint32_t distinct = 0;
            // pass 1: insert (worker -> first epoch, count) and mark the bitmap
            for (uint32_t r = 0; r < rounds; ++r) {
                const uint32_t e = r * 32 + lane;
                uint32_t w = kNone;
                if (e < E) {
                    const uint32_t p = T[e * 32 + s];
                    if (p < part.P) {
                        const uint32_t ww = part.worker_of(p);
                        if (ww >= part.wbegin && ww < part.wend) w = ww - part.wbegin;
                    }
                }
                const uint32_t m = __match_any_sync(0xffffffffu, w);
                const bool leader = (__ffs(m) - 1) == (int)lane;
                bool fresh = false;
                if (w != kNone && leader) {
                    uint32_t slot = hash_slot(w, mask);
                    while (true) {
                        const uint32_t old = atomicCAS(&keys[slot], kNone, w);
                        if (old == kNone) {
                            vals[slot] = (e << 16) | __popc(m);
                            fresh = true;
                            break;
                        }
                        if (old == w) {
                            vals[slot] += __popc(m);
                            break;
                        }
                        slot = (slot + 1) & mask;
                    }
                    if (fresh) atomicOr(&bm[w >> 5], 1u << (w & 31));
                }
                distinct += __popc(__ballot_sync(0xffffffffu, fresh));
                __syncwarp();
            }
            // bitmap prefix popcounts -> rank(w) = pre[w>>5] + popc(bm[w>>5] & below)
            {
                const uint32_t per = (nw_words + 31) / 32;
                const uint32_t b0 = lane * per;
                uint32_t local = 0;
                for (uint32_t t = 0; t < per; ++t)
                    if (b0 + t < nw_words) local += __popc(bm[b0 + t]);
                uint32_t incl = local;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
                    if ((int)lane >= o) incl += v;
                }
                uint32_t run = incl - local;
                for (uint32_t t = 0; t < per; ++t)
                    if (b0 + t < nw_words) {
                        pre[b0 + t] = run;
                        run += __popc(bm[b0 + t]);
                    }
            }
            __syncwarp();
            // pass 2: emit info in place
            for (uint32_t r = 0; r < rounds; ++r) {
                const uint32_t e = r * 32 + lane;
                if (e < E) {
                    const uint32_t p = T[e * 32 + s];
                    uint32_t out = 0;
                    if (p < part.P) {
                        const uint32_t ww = part.worker_of(p);
                        if (ww >= part.wbegin && ww < part.wend) {
                            const uint32_t w = ww - part.wbegin;
                            uint32_t slot = hash_slot(w, mask);
                            while (keys[slot] != w) slot = (slot + 1) & mask;
                            const uint32_t v = vals[slot];
                            if ((v >> 16) == e) {
                                const uint32_t rank =
                                    pre[w >> 5] + __popc(bm[w >> 5] & ((1u << (w & 31)) - 1u));
                                out = ((v & 0xFFFFu) << 16) | rank;
                            }
                        }
                    }
                    T[e * 32 + s] = out;
                }
            }
            __syncwarp();
            for (uint32_t t = lane; t < hs; t += 32) keys[t] = kNone;
            for (uint32_t t = lane; t < nw_words; t += 32) bm[t] = 0;
            if (lane == 0) pair_count[k0 + s] = distinct;
            __syncwarp();
        }
        __syncthreads();
        for (uint32_t idx = threadIdx.x; idx < E * 32; idx += blockDim.x) {
            const uint32_t e = idx >> 5, l = idx & 31;
            if (k0 + l < F) info[(size_t)e * pitch16(F) + k0 + l] = T[idx];
        }
    }
}

int sample_pass_config(const Part& part, uint32_t* hs, uint32_t* nw_words, uint32_t* warps,
                       size_t* smem) {
    const uint32_t nloc = part.wend - part.wbegin;
    uint32_t d = part.E < nloc ? part.E : nloc;
    uint32_t h = 32;
    while (h < 2 * d) h <<= 1;
    *hs = h;
    *nw_words = (nloc + 31) / 32;
    for (uint32_t wp = 8; wp >= 1; wp >>= 1) {
        const size_t bytes =
            (size_t)part.E * 32 * 4 + (size_t)wp * (2 * (size_t)h + 2 * (size_t)*nw_words) * 4;
        if (bytes <= 200 * 1024) {
            *warps = wp;
            *smem = bytes;
            return 0;
        }
    }
    return -1;
}

void launch_sample_pass(cudaStream_t s, const Part& part, uint32_t* info, uint32_t* pair_count,
                        uint32_t hs, uint32_t nw_words, uint32_t warps, size_t smem) {
    // per-device attribute; cheap and idempotent
    allow_smem(sample_pass_kernel, 
                         200 * 1024);
    const unsigned grid = grid_for(((uint64_t)part.F + 31) / 32, 1, 148u * 8u);
    sample_pass_kernel<<<grid, warps * 32, smem, s>>>(part, info, pair_count, hs, nw_words);
}

}  // namespace clairplan
