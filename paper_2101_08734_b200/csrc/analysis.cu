// Analysis reuse: the reference's analysis / acceptance checks consume the
// access counts (access.cpp:90-116); here the counts never leave the device.
//   clairplan_count_histogram       FrequencyHistogram of one worker's counts on a built plan
//   clairplan_monte_carlo_histogram monte_carlo_histogram (analysis.cpp:84-96): worker 0 of the
//                                   B = N, drop_last = false partition, bucketed on the device
//   clairplan_count_extremes        per sample the largest and smallest count over all workers:
//                                   everything the Lemma-1 property suite inspects
//                                   (acceptance.cpp:98-158 — "the other workers' minimum"
//                                   after removing one holder of the maximum is the minimum)
#include "plan_impl.h"

namespace clairplan {

__global__ void count_bucket_kernel(const uint32_t* __restrict__ counts, uint32_t F, uint32_t maxc,
                                    unsigned long long* __restrict__ buckets) {
    extern __shared__ unsigned long long sb[];
    for (uint32_t c = threadIdx.x; c <= maxc; c += blockDim.x) sb[c] = 0;
    __syncthreads();
    for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < F; k += gridDim.x * blockDim.x)
        atomicAdd(&sb[min(counts[k], maxc)], 1ull);
    __syncthreads();
    for (uint32_t c = threadIdx.x; c <= maxc; c += blockDim.x)
        if (sb[c]) atomicAdd(&buckets[c], sb[c]);
}

__global__ void extremes_kernel(const uint32_t* __restrict__ counts, uint32_t F, int first,
                                uint32_t* __restrict__ hi, uint32_t* __restrict__ lo) {
    for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < F; k += gridDim.x * blockDim.x) {
        const uint32_t c = counts[k];
        hi[k] = first ? c : max(hi[k], c);
        lo[k] = first ? c : min(lo[k], c);
    }
}

// counts of worker w (its stream on the device) into d_counts[F]
static int worker_counts_dev(clairplan_plan* p, uint32_t w, uint32_t* d_counts) {
    const uint64_t a = p->part.stream_offset(w), b = p->part.stream_offset(w + 1);
    CK(cudaMemsetAsync(d_counts, 0, (size_t)p->part.F * 4, p->stream));
    if (b > a) launch_stream_hist(p->stream, p->stream_buf.get<uint32_t>() + a, b - a, d_counts);
    return 0;
}

static int plan_for_counts(const clairplan_config* cfg, uint32_t wb, uint32_t we, clairplan_t* out) {
    clairplan_config c = *cfg;
    c.num_classes = 0;
    c.worker_begin = wb;
    c.worker_end = we;
    if (int rc = clairplan_create(&c, out)) return rc;
    if (int rc = clairplan_build(*out)) {
        clairplan_destroy(*out);
        *out = nullptr;
        return rc;
    }
    return 0;
}

}  // namespace clairplan

extern "C" {

int clairplan_count_histogram(clairplan_t p, uint32_t worker, uint32_t max_count, uint64_t* buckets) {
    if (!p || !p->built || p->generic) return fail(CLAIRPLAN_EINVAL, "plan not built");
    if (!buckets) return fail(CLAIRPLAN_EINVAL, "null argument");
    if (worker < p->part.wbegin || worker >= p->part.wend) return fail(CLAIRPLAN_EINVAL, "worker not in plan");
    if (max_count > 65535) return fail(CLAIRPLAN_EINVAL, "max_count too large");
    CK(cudaSetDevice(p->device));
    DevBuf cnt, hb;
    if (!cnt.ensure((size_t)p->part.F * 4) || !hb.ensure(((size_t)max_count + 1) * 8))
        return fail(CLAIRPLAN_ENOMEM, "device allocation failed");
    if (int rc = worker_counts_dev(p, worker, cnt.get<uint32_t>())) return rc;
    CK(cudaMemsetAsync(hb.p, 0, ((size_t)max_count + 1) * 8, p->stream));
    const size_t smem = ((size_t)max_count + 1) * 8;
    CK(allow_smem(count_bucket_kernel, (int)smem));
    count_bucket_kernel<<<grid_for(p->part.F, kThreads, 148u * 4u), kThreads, smem, p->stream>>>(
        cnt.get<uint32_t>(), p->part.F, max_count, hb.get<unsigned long long>());
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(buckets, hb.p, ((size_t)max_count + 1) * 8, cudaMemcpyDeviceToHost, p->stream));
    CK(cudaStreamSynchronize(p->stream));
    return 0;
}

int clairplan_monte_carlo_histogram(uint64_t seed, uint32_t workers, uint32_t epochs, uint32_t samples,
                                    uint64_t* buckets, int device) {
    clairplan_config c{};
    c.seed = seed;
    c.samples = samples;
    c.num_workers = workers;
    c.global_batch = workers;  // one sample per worker per iteration (analysis.cpp:87-90)
    c.epochs = epochs;
    c.drop_last = 0;
    c.device = device;
    if (int rc = clairplan_validate(&c)) return rc;
    clairplan_t p = nullptr;
    if (int rc = plan_for_counts(&c, 0, 1, &p)) return rc;
    const int rc = clairplan_count_histogram(p, 0, epochs, buckets);
    clairplan_destroy(p);
    return rc;
}

int clairplan_count_extremes(const clairplan_config* cfg, uint32_t* hi, uint32_t* lo) {
    if (!cfg || !hi || !lo) return fail(CLAIRPLAN_EINVAL, "null argument");
    if (int rc = clairplan_validate(cfg)) return rc;
    clairplan_t p = nullptr;
    if (int rc = plan_for_counts(cfg, 0, cfg->num_workers, &p)) return rc;
    const uint32_t F = cfg->samples;
    DevBuf cnt, ext;
    int rc = 0;
    if (!cnt.ensure((size_t)F * 4) || !ext.ensure((size_t)F * 8)) {
        rc = fail(CLAIRPLAN_ENOMEM, "device allocation failed");
    } else {
        for (uint32_t w = 0; w < cfg->num_workers && !rc; ++w) {
            rc = worker_counts_dev(p, w, cnt.get<uint32_t>());
            if (!rc)
                extremes_kernel<<<grid_for(F, kThreads), kThreads, 0, p->stream>>>(
                    cnt.get<uint32_t>(), F, w == 0, ext.get<uint32_t>(), ext.get<uint32_t>() + F);
        }
        if (!rc && (cudaMemcpyAsync(hi, ext.p, (size_t)F * 4, cudaMemcpyDeviceToHost, p->stream) != cudaSuccess ||
                    cudaMemcpyAsync(lo, ext.get<uint32_t>() + F, (size_t)F * 4, cudaMemcpyDeviceToHost,
                                    p->stream) != cudaSuccess ||
                    cudaStreamSynchronize(p->stream) != cudaSuccess))
            rc = fail(CLAIRPLAN_ECUDA, "count extremes copy failed");
    }
    clairplan_destroy(p);
    return rc;
}

}  // extern "C"
