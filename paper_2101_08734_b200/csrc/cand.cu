// K4b: per-worker candidate lists in first-access order (policies.cpp:151-156).
//
// A (worker, sample) pair is a candidate iff the worker reads the sample (count > 0).  The
// pair's first access is the stream entry whose info word (sample pass) is non-zero.  A
// worker's stream is a sequence of epoch segments; segment (w, e) is contiguous in the
// worker-major stream, and every info lookup of that segment hits row e of info[E][F] — CTAs
// are ordered epoch-major so row e stays L2-resident while its segments stream through.
//   seg_count : number of first accesses per segment           -> segcnt[w*E + e]
//   seg_write : cand_k / cand_info compacted in stream order at seg_off[w*E + e]
#include "internal.h"

namespace clairplan {

__global__ void __launch_bounds__(kThreads) seg_count_kernel(Part part,
                                                              const uint32_t* __restrict__ stream,
                                                              const uint32_t* __restrict__ info,
                                                              uint32_t* __restrict__ segcnt) {
    __shared__ uint32_t wsum[kThreads / 32];
    const uint32_t nloc = part.wend - part.wbegin;
    const uint64_t nseg = (uint64_t)nloc * part.E;
    for (uint64_t b = blockIdx.x; b < nseg; b += gridDim.x) {
        const uint32_t e = (uint32_t)(b / nloc), wl = (uint32_t)(b % nloc);
        const uint32_t w = part.wbegin + wl;
        const uint64_t Le = part.epoch_len(w);
        const uint64_t g0 = part.stream_offset(w) + (uint64_t)e * Le;
        const uint32_t* row = info + (size_t)e * part.Fp;
        uint32_t c = 0;
        for (uint64_t t = threadIdx.x; t < Le; t += blockDim.x) c += row[stream[g0 + t]] != 0;
        c = warp_sum(c);
        if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = c;
        __syncthreads();
        if (threadIdx.x == 0) {
            uint32_t s = 0;
            for (int i = 0; i < kThreads / 32; ++i) s += wsum[i];
            segcnt[(uint64_t)wl * part.E + e] = s;
        }
        __syncthreads();
    }
}

__global__ void __launch_bounds__(kThreads) seg_write_kernel(Part part,
                                                              const uint32_t* __restrict__ stream,
                                                              const uint32_t* __restrict__ info,
                                                              const uint64_t* __restrict__ seg_off,
                                                              uint32_t* __restrict__ cand_k,
                                                              uint32_t* __restrict__ cand_info) {
    __shared__ uint32_t wsum[kThreads / 32];
    const uint32_t nloc = part.wend - part.wbegin;
    const uint64_t nseg = (uint64_t)nloc * part.E;
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (uint64_t b = blockIdx.x; b < nseg; b += gridDim.x) {
        const uint32_t e = (uint32_t)(b / nloc), wl = (uint32_t)(b % nloc);
        const uint32_t w = part.wbegin + wl;
        const uint64_t Le = part.epoch_len(w);
        const uint64_t g0 = part.stream_offset(w) + (uint64_t)e * Le;
        const uint32_t* row = info + (size_t)e * part.Fp;
        uint64_t out = seg_off[(uint64_t)wl * part.E + e];
        for (uint64_t t0 = 0; t0 < Le; t0 += blockDim.x) {
            const uint64_t t = t0 + threadIdx.x;
            uint32_t k = 0, inf = 0;
            if (t < Le) {
                k = stream[g0 + t];
                inf = row[k];
            }
            const uint32_t bal = __ballot_sync(0xffffffffu, inf != 0);
            if (lane == 0) wsum[warp] = __popc(bal);
            __syncthreads();
            uint32_t below = 0, tot = 0;
#pragma unroll
            for (int i = 0; i < kThreads / 32; ++i) {
                const uint32_t v = wsum[i];
                below += (i < (int)warp) ? v : 0;
                tot += v;
            }
            if (inf != 0) {
                const uint64_t pos = out + below + __popc(bal & lanemask_lt());
                cand_k[pos] = k;
                cand_info[pos] = inf;
            }
            out += tot;
            __syncthreads();
        }
    }
}

// per-worker candidate segment [begin, begin+len) from the (w, e) segment offsets
__global__ void worker_segments_kernel(const uint64_t* __restrict__ seg_off, uint32_t nloc,
                                       uint32_t E, uint64_t* __restrict__ wbegin,
                                       uint64_t* __restrict__ wlen) {
    for (uint32_t w = blockIdx.x * blockDim.x + threadIdx.x; w < nloc; w += gridDim.x * blockDim.x) {
        const uint64_t a = seg_off[(uint64_t)w * E], b = seg_off[(uint64_t)(w + 1) * E];
        wbegin[w] = a;
        wlen[w] = b - a;
    }
}

void launch_seg_count(cudaStream_t s, const Part& part, const uint32_t* stream,
                      const uint32_t* info, uint32_t* segcnt) {
    const uint64_t nseg = (uint64_t)(part.wend - part.wbegin) * part.E;
    seg_count_kernel<<<grid_for(nseg, 1, 148u * 32u), kThreads, 0, s>>>(part, stream, info, segcnt);
}

void launch_seg_write(cudaStream_t s, const Part& part, const uint32_t* stream,
                      const uint32_t* info, const uint64_t* seg_off, uint32_t* cand_k,
                      uint32_t* cand_info) {
    const uint64_t nseg = (uint64_t)(part.wend - part.wbegin) * part.E;
    seg_write_kernel<<<grid_for(nseg, 1, 148u * 32u), kThreads, 0, s>>>(part, stream, info,
                                                                        seg_off, cand_k, cand_info);
}

void launch_worker_segments(cudaStream_t s, const uint64_t* seg_off, uint32_t nloc, uint32_t E,
                            uint64_t* wbegin, uint64_t* wlen) {
    worker_segments_kernel<<<grid_for(nloc, kThreads), kThreads, 0, s>>>(seg_off, nloc, E, wbegin,
                                                                         wlen);
}

}  // namespace clairplan
