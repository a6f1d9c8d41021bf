// Multi-GPU building blocks: epoch-range streams are exchanged with one NCCL
// all-to-all; the receiving rank re-lays them out into its worker-major streams and rebuilds
// the inverse permutations restricted to its workers.
//
//   stream_relayout  recv [source r][local worker w][epoch e of r][Le(w)]  (all-to-all output)
//                    -> stream [w][e][Le(w)]  (the handle's layout, build_access_streams order,
//                    access.cpp:59-78)
//   stream_inv       inv[e][k] = position of k in epoch e's permutation for every entry of the
//                    handle's streams (batch_slice geometry, access.cpp:14-39); other samples
//                    keep kNone (they belong to other ranks' workers)
#include "internal.h"

namespace clairplan {

// one CTA column per (source, worker) chunk, blockIdx.y splits the chunk
__global__ void __launch_bounds__(kThreads) stream_relayout_kernel(Part part, EpochSplit es,
                                                                   const uint32_t* __restrict__ recv,
                                                                   uint32_t* __restrict__ stream) {
    const uint32_t nloc = part.wend - part.wbegin;
    const uint32_t r = blockIdx.x / nloc, wl = blockIdx.x - r * nloc;
    const uint32_t w = part.wbegin + wl;
    const uint64_t p0 = part.prefix_len(part.wbegin);
    const uint64_t lloc = part.prefix_len(part.wend) - p0;  // local entries per epoch
    const uint32_t e0 = es.eb[r], ne = es.eb[r + 1] - e0;
    const uint64_t Le = part.epoch_len(w);
    const uint64_t n = (uint64_t)ne * Le;
    const uint32_t* src = recv + (uint64_t)e0 * lloc + (uint64_t)ne * (part.prefix_len(w) - p0);
    uint32_t* dst = stream + part.stream_offset(w) + (uint64_t)e0 * Le;
    const uint64_t per = (n + gridDim.y - 1) / gridDim.y;
    const uint64_t a = per * blockIdx.y, b = a + per < n ? a + per : n;
    if (a >= b) return;
    const bool vec = ((((uintptr_t)(src + a)) | ((uintptr_t)(dst + a))) & 15) == 0;
    if (vec) {
        const uint64_t nv = (b - a) / 4;
        const uint4* s4 = reinterpret_cast<const uint4*>(src + a);
        uint4* d4 = reinterpret_cast<uint4*>(dst + a);
        for (uint64_t i = threadIdx.x; i < nv; i += blockDim.x) __stcs(d4 + i, __ldcs(s4 + i));
        for (uint64_t i = a + nv * 4 + threadIdx.x; i < b; i += blockDim.x) dst[i] = src[i];
    } else {
        for (uint64_t i = a + threadIdx.x; i < b; i += blockDim.x) dst[i] = __ldcs(src + i);
    }
}

// one warp per (worker, epoch) segment, lanes over the segment's entries
__global__ void __launch_bounds__(kThreads) stream_inv_kernel(Part part, const uint32_t* __restrict__ stream,
                                                              uint32_t* __restrict__ inv) {
    const uint32_t E = part.E, F = part.F, nloc = part.wend - part.wbegin;
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t nseg = (uint64_t)nloc * E;
    for (uint64_t sg = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; sg < nseg;
         sg += ((uint64_t)gridDim.x * blockDim.x) >> 5) {
        const uint32_t e = (uint32_t)(sg / nloc), wl = (uint32_t)(sg - (uint64_t)e * nloc);
        const uint32_t w = part.wbegin + wl;
        const uint32_t L = (uint32_t)part.len(w);
        const FastDiv& dl = w < part.extra ? part.dFull1 : part.dFull0;
        const uint32_t fb = (uint32_t)(w * part.base + (w < part.extra ? w : part.extra));
        const uint32_t tb = (uint32_t)(w * part.tbase + (w < part.textra ? w : part.textra));
        const uint32_t nfull = (uint32_t)(part.full * L);
        const uint32_t Le = (uint32_t)part.epoch_len(w);
        const uint32_t* seg = stream + part.stream_offset(w) + (uint64_t)e * Le;
        uint32_t* row = inv + (size_t)e * F;
        for (uint32_t t = lane; t < Le; t += 32) {
            uint32_t pos;
            if (t < nfull) {
                const uint32_t h = dl.div(t);
                pos = h * part.B + fb + (t - h * L);
            } else {
                pos = (uint32_t)(part.full * part.B) + tb + (t - nfull);
            }
            row[__ldcs(seg + t)] = pos;
        }
    }
}

void launch_stream_relayout(cudaStream_t s, const Part& part, const EpochSplit& es,
                            const uint32_t* recv, uint32_t* stream) {
    const uint32_t nloc = part.wend - part.wbegin;
    dim3 grid(nloc * es.G, std::max<uint32_t>(1, (148u * 8u) / std::max<uint32_t>(1, nloc * es.G)));
    stream_relayout_kernel<<<grid, kThreads, 0, s>>>(part, es, recv, stream);
}

void launch_stream_inv(cudaStream_t s, const Part& part, const uint32_t* stream, uint32_t* inv) {
    const uint64_t nseg = (uint64_t)(part.wend - part.wbegin) * part.E;
    stream_inv_kernel<<<grid_for(nseg * 32, kThreads, 148u * 64u), kThreads, 0, s>>>(part, stream, inv);
}

}  // namespace clairplan
