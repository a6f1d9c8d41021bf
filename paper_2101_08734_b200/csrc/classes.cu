// K7/K8 helpers: tier bookkeeping, prefetch-order class lists, holder CSR.
#include "internal.h"

namespace clairplan {

// sorted_size[i] = sizes[cand_k[order[i]]]  (candidates in tier order, policies.cpp:157-161)
__global__ void gather_sizes_kernel(const uint32_t* __restrict__ order,
                                    const uint32_t* __restrict__ cand_k,
                                    const double* __restrict__ sizes, uint64_t n,
                                    double* __restrict__ out) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x)
        out[i] = sizes[cand_k[order[i]]];
}

// sort key "count descending": (maxc - count) so that a stable ascending pass is the
// reference's stable_sort by count desc with first-access order preserved inside counts
__global__ void count_keys_kernel(const uint32_t* __restrict__ cand_info, uint64_t n,
                                  uint32_t maxc, uint32_t* __restrict__ keys) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x)
        keys[i] = maxc - (cand_info[i] >> 16);
}

// class of pass j: sorted element i taken -> cls[order[i]] = j  (only if not yet assigned)
__global__ void apply_pass_kernel(const uint8_t* __restrict__ taken, uint64_t n,
                                  const uint32_t* __restrict__ seq_to_sorted,
                                  const uint32_t* __restrict__ order, uint8_t cls,
                                  uint8_t* __restrict__ cand_cls) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        if (!taken[i]) continue;
        const uint32_t si = seq_to_sorted ? seq_to_sorted[i] : (uint32_t)i;
        cand_cls[order ? order[si] : si] = cls;
    }
}

// rejects of pass j in tier order: key = taken (0 first) for a stable partition
__global__ void reject_keys_kernel(const uint8_t* __restrict__ taken, uint64_t n,
                                   const uint32_t* __restrict__ seq_to_sorted,
                                   uint32_t* __restrict__ keys, uint32_t* __restrict__ vals) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        keys[i] = taken[i];
        vals[i] = seq_to_sorted ? seq_to_sorted[i] : (uint32_t)i;
    }
}

__global__ void gather_seq_sizes_kernel(const uint32_t* __restrict__ idx,
                                        const double* __restrict__ sorted_size,
                                        const uint64_t* __restrict__ seg_begin,
                                        const uint64_t* __restrict__ seg_len, uint32_t nseg,
                                        double* __restrict__ out) {
    // elements outside segments are ignored; iterate segment-by-segment
    for (uint32_t seg = blockIdx.x; seg < nseg; seg += gridDim.x) {
        const uint64_t b = seg_begin[seg], L = seg_len[seg];
        for (uint64_t i = threadIdx.x; i < L; i += blockDim.x) out[b + i] = sorted_size[idx[b + i]];
    }
}

// class digit: classes 1..J -> 0..J-1, unassigned -> J (after every class list)
__global__ void class_keys_kernel(const uint8_t* __restrict__ cand_cls, uint64_t n, uint32_t J,
                                  uint32_t* __restrict__ keys) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t c = cand_cls[i];
        keys[i] = c ? c - 1 : J;
    }
}

// holder record of every candidate at its sample-major pair slot (build_index order:
// per sample, workers ascending).  cls == 0 marks an unassigned pair.
__global__ void holder_scatter_kernel(const uint32_t* __restrict__ cand_k,
                                      const uint32_t* __restrict__ cand_info,
                                      const uint8_t* __restrict__ cand_cls,
                                      const uint32_t* __restrict__ dest,
                                      const uint64_t* __restrict__ wbegin,
                                      const uint64_t* __restrict__ wlen,
                                      const uint64_t* __restrict__ class_start, uint32_t J,
                                      uint32_t nloc, uint32_t worker0,
                                      const uint64_t* __restrict__ pair_off,
                                      uint32_t* __restrict__ holders) {
    for (uint32_t wl = blockIdx.x; wl < nloc; wl += gridDim.x) {
        const uint64_t b = wbegin[wl], L = wlen[wl];
        for (uint64_t i = threadIdx.x; i < L; i += blockDim.x) {
            const uint64_t c = b + i;
            const uint32_t k = cand_k[c];
            const uint32_t rank = cand_info[c] & 0xFFFFu;
            const uint32_t cls = cand_cls[c];
            const uint64_t slot = pair_off[k] + rank;
            uint32_t pos = 0;
            if (cls) pos = (uint32_t)(dest[c] - class_start[(uint64_t)wl * (J + 1) + cls - 1]);
            holders[3 * slot + 0] = worker0 + wl;
            holders[3 * slot + 1] = cls;
            holders[3 * slot + 2] = pos;
        }
    }
}

// per sample: number of assigned pairs in its pair range
__global__ void holder_count_kernel(const uint64_t* __restrict__ pair_off, uint32_t F,
                                    const uint32_t* __restrict__ tmp, uint32_t* __restrict__ cnt) {
    for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < F; k += gridDim.x * blockDim.x) {
        uint32_t c = 0;
        for (uint64_t s = pair_off[k]; s < pair_off[k + 1]; ++s) c += tmp[3 * s + 1] != 0;
        cnt[k] = c;
    }
}

__global__ void holder_compact_kernel(const uint64_t* __restrict__ pair_off, uint32_t F,
                                      const uint32_t* __restrict__ tmp,
                                      const uint64_t* __restrict__ hoff,
                                      uint32_t* __restrict__ holders) {
    for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < F; k += gridDim.x * blockDim.x) {
        uint64_t o = hoff[k];
        for (uint64_t s = pair_off[k]; s < pair_off[k + 1]; ++s) {
            if (tmp[3 * s + 1] == 0) continue;
            holders[3 * o + 0] = tmp[3 * s + 0];
            holders[3 * o + 1] = tmp[3 * s + 1];
            holders[3 * o + 2] = tmp[3 * s + 2];
            ++o;
        }
    }
}

__global__ void stream_hist_kernel(const uint32_t* __restrict__ st, uint64_t n,
                                   uint32_t* __restrict__ counts) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x)
        atomicAdd(&counts[st[i]], 1u);
}

void launch_stream_hist(cudaStream_t s, const uint32_t* st, uint64_t n, uint32_t* counts) {
    stream_hist_kernel<<<grid_for(n, kThreads), kThreads, 0, s>>>(st, n, counts);
}

void launch_gather_sizes(cudaStream_t s, const uint32_t* order, const uint32_t* cand_k,
                         const double* sizes, uint64_t n, double* out) {
    gather_sizes_kernel<<<grid_for(n, kThreads), kThreads, 0, s>>>(order, cand_k, sizes, n, out);
}
void launch_count_keys(cudaStream_t s, const uint32_t* cand_info, uint64_t n, uint32_t maxc,
                       uint32_t* keys) {
    count_keys_kernel<<<grid_for(n, kThreads), kThreads, 0, s>>>(cand_info, n, maxc, keys);
}
void launch_apply_pass(cudaStream_t s, const uint8_t* taken, uint64_t n,
                       const uint32_t* seq_to_sorted, const uint32_t* order, uint8_t cls,
                       uint8_t* cand_cls) {
    apply_pass_kernel<<<grid_for(n, kThreads), kThreads, 0, s>>>(taken, n, seq_to_sorted, order,
                                                                 cls, cand_cls);
}
void launch_reject_keys(cudaStream_t s, const uint8_t* taken, uint64_t n,
                        const uint32_t* seq_to_sorted, uint32_t* keys, uint32_t* vals) {
    reject_keys_kernel<<<grid_for(n, kThreads), kThreads, 0, s>>>(taken, n, seq_to_sorted, keys,
                                                                  vals);
}
void launch_gather_seq_sizes(cudaStream_t s, const uint32_t* idx, const double* sorted_size,
                             const uint64_t* seg_begin, const uint64_t* seg_len, uint32_t nseg,
                             double* out) {
    gather_seq_sizes_kernel<<<grid_for((uint64_t)nseg, 1, 148u * 16u), kThreads, 0, s>>>(
        idx, sorted_size, seg_begin, seg_len, nseg, out);
}
void launch_class_keys(cudaStream_t s, const uint8_t* cand_cls, uint64_t n, uint32_t J,
                       uint32_t* keys) {
    class_keys_kernel<<<grid_for(n, kThreads), kThreads, 0, s>>>(cand_cls, n, J, keys);
}
void launch_holder_scatter(cudaStream_t s, const uint32_t* cand_k, const uint32_t* cand_info,
                           const uint8_t* cand_cls, const uint32_t* dest, const uint64_t* wbegin,
                           const uint64_t* wlen, const uint64_t* class_start, uint32_t J,
                           uint32_t nloc, uint32_t worker0, const uint64_t* pair_off,
                           uint32_t* holders) {
    holder_scatter_kernel<<<grid_for(nloc, 1, 148u * 16u), kThreads, 0, s>>>(
        cand_k, cand_info, cand_cls, dest, wbegin, wlen, class_start, J, nloc, worker0, pair_off,
        holders);
}
void launch_holder_count(cudaStream_t s, const uint64_t* pair_off, uint32_t F, const uint32_t* tmp,
                         uint32_t* cnt) {
    holder_count_kernel<<<grid_for(F, kThreads), kThreads, 0, s>>>(pair_off, F, tmp, cnt);
}
void launch_holder_compact(cudaStream_t s, const uint64_t* pair_off, uint32_t F,
                           const uint32_t* tmp, const uint64_t* hoff, uint32_t* holders) {
    holder_compact_kernel<<<grid_for(F, kThreads), kThreads, 0, s>>>(pair_off, F, tmp, hoff,
                                                                     holders);
}

}  // namespace clairplan
