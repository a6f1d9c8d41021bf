// Plan wire format: a versioned, self-describing binary image of one handle's
// plan — streams, per-(worker, class) list bounds, class lists (prefetch orders), holder CSR —
// for files and for shipping plans between processes / nodes (the paper's middleware
// all-gathers the access information at setup; the reference has no plan
// serialization at all, clairsim_main.cpp:88-151 prints summaries).
//
// Layout (little-endian, every section 16-B aligned):
//   clairplan_wire_header (256 B) | capacities f64[J] | streams u32[A]
//   | class bounds u64[2 * nloc * J] (offset into the class-list section, length)
//   | class lists u32[sum of lengths] | holder offsets u64[F + 1] | holders u32[3 H]
// Every section carries a 64-bit position-keyed checksum computed on the device before the
// copy: sum over i of mix64(key_s + i * golden) ^ word_i (mod 2^64) for 32-bit words, a
// "checksum of the words at their positions" that any order of summation reproduces.
#include <cstring>

#include "plan_impl.h"

static_assert(sizeof(clairplan_wire_header) == 256, "wire header is 256 bytes");

namespace clairplan {

__global__ void wire_sum_kernel(const uint32_t* __restrict__ w, uint64_t n, uint64_t key,
                                unsigned long long* __restrict__ out) {
    unsigned long long acc = 0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x)
        acc += mix64(key + i * kGolden) ^ (uint64_t)w[i];
    acc = warp_sum(acc);
    if ((threadIdx.x & 31) == 0 && acc) atomicAdd(out, acc);
}

// holder records of a shard summed at their positions in the merged (all-shard) CSR:
// record r of sample k sits at starts[k] + (r - own_offset[k])
__global__ void wire_holder_sum_kernel(const uint32_t* __restrict__ hold, const uint64_t* __restrict__ hoff,
                                       const uint64_t* __restrict__ starts, uint32_t F, uint64_t key,
                                       unsigned long long* __restrict__ out) {
    unsigned long long acc = 0;
    for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < F; k += gridDim.x * blockDim.x) {
        const uint64_t a = hoff[k], b = hoff[k + 1], g = starts[k];
        for (uint64_t r = a; r < b; ++r)
            for (uint32_t c = 0; c < 3; ++c)
                acc += mix64(key + (3 * (g + r - a) + c) * kGolden) ^ (uint64_t)hold[3 * r + c];
    }
    acc = warp_sum(acc);
    if ((threadIdx.x & 31) == 0 && acc) atomicAdd(out, acc);
}

// a section of `words` 32-bit words starting at word position `base` of the merged section
__global__ void wire_sum_at_kernel(const uint32_t* __restrict__ w, uint64_t n, uint64_t base,
                                   uint64_t key, unsigned long long* __restrict__ out) {
    unsigned long long acc = 0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x)
        acc += mix64(key + (base + i) * kGolden) ^ (uint64_t)w[i];
    acc = warp_sum(acc);
    if ((threadIdx.x & 31) == 0 && acc) atomicAdd(out, acc);
}

static uint64_t align16(uint64_t x) { return (x + 15) & ~15ull; }

struct WireLayout {
    uint64_t caps, streams, bounds, lists, hoff, holders, total;
    uint64_t ncl;  // class-list entries
};

static WireLayout wire_layout(const clairplan_plan* p) {
    const uint32_t J = p->cfg.num_classes, nloc = p->nloc;
    WireLayout L{};
    uint64_t ncl = 0;
    for (uint32_t w = 0; w < nloc; ++w)
        for (uint32_t j = 0; j < J; ++j) ncl += p->class_len_h[(size_t)w * (J + 1) + j];
    L.ncl = ncl;
    L.caps = align16(sizeof(clairplan_wire_header));
    L.streams = align16(L.caps + 8ull * J);
    L.bounds = align16(L.streams + 4ull * p->A);
    L.lists = align16(L.bounds + 16ull * nloc * J);
    L.hoff = align16(L.lists + 4ull * ncl);
    L.holders = align16(L.hoff + 8ull * ((uint64_t)p->part.F + 1));
    L.total = align16(L.holders + 12ull * p->H);
    return L;
}

}  // namespace clairplan

extern "C" {

int clairplan_wire_size(clairplan_t p, uint64_t* bytes) {
    if (!p || !p->built || p->generic) return fail(CLAIRPLAN_EINVAL, "plan not built");
    if (!bytes) return fail(CLAIRPLAN_EINVAL, "null argument");
    *bytes = wire_layout(p).total;
    return 0;
}

int clairplan_wire_write(clairplan_t p, void* out, uint64_t cap) {
    if (!p || !p->built || p->generic) return fail(CLAIRPLAN_EINVAL, "plan not built");
    if (!out) return fail(CLAIRPLAN_EINVAL, "null argument");
    const WireLayout L = wire_layout(p);
    if (cap < L.total) return fail(CLAIRPLAN_ERANGE, "output buffer too small");
    CK(cudaSetDevice(p->device));
    cudaStream_t s = p->stream;
    char* o = static_cast<char*>(out);
    memset(o, 0, L.total);
    const uint32_t J = p->cfg.num_classes, nloc = p->nloc, F = p->part.F;
    clairplan_wire_header h{};
    memcpy(h.magic, "CLPLAN\0\1", 8);
    h.version = CLAIRPLAN_WIRE_VERSION;
    h.header_bytes = sizeof(clairplan_wire_header);
    h.seed = p->cfg.seed;
    h.samples = F;
    h.num_workers = p->part.N;
    h.global_batch = p->part.B;
    h.epochs = p->part.E;
    h.drop_last = p->part.drop_last;
    h.num_classes = J;
    h.worker_begin = p->part.wbegin;
    h.worker_end = p->part.wend;
    h.accesses = p->A;
    h.class_entries = L.ncl;
    h.holders = p->H;
    h.off_caps = L.caps;
    h.off_streams = L.streams;
    h.off_class_bounds = L.bounds;
    h.off_class_lists = L.lists;
    h.off_holder_offsets = L.hoff;
    h.off_holders = L.holders;
    h.total_bytes = L.total;
    // device-side section checksums (32-bit words at their positions)
    DevBuf sums;
    if (!sums.ensure(8 * 6)) return fail(CLAIRPLAN_ENOMEM, "device allocation failed");
    CK(cudaMemsetAsync(sums.p, 0, 8 * 6, s));
    unsigned long long* ds = sums.get<unsigned long long>();
    auto dsum = [&](const void* d, uint64_t words, int sec) {
        if (words)
            wire_sum_kernel<<<grid_for(words, kThreads, 148u * 8u), kThreads, 0, s>>>(
                static_cast<const uint32_t*>(d), words, (uint64_t)sec << 56, ds + sec);
    };
    dsum(p->stream_buf.get<uint32_t>(), p->A, 1);
    dsum(p->holder_off_dev, 2 * ((uint64_t)F + 1), 4);
    if (p->H) dsum(p->holders_dev, 3 * p->H, 5);
    // sections
    if (J) memcpy(o + L.caps, p->caps.data(), 8ull * J);
    CK(cudaMemcpyAsync(o + L.streams, p->stream_buf.p, 4ull * p->A, cudaMemcpyDeviceToHost, s));
    uint64_t* bounds = reinterpret_cast<uint64_t*>(o + L.bounds);
    uint64_t run = 0;
    for (uint32_t w = 0; w < nloc; ++w)
        for (uint32_t j = 0; j < J; ++j) {
            const uint64_t n = p->class_len_h[(size_t)w * (J + 1) + j];
            bounds[2 * ((uint64_t)w * J + j)] = run;
            bounds[2 * ((uint64_t)w * J + j) + 1] = n;
            run += n;
        }
    if (int rc = clairplan_export_class_lists_async(p, reinterpret_cast<uint32_t*>(o + L.lists), L.ncl))
        return rc;
    CK(cudaMemcpyAsync(o + L.hoff, p->holder_off_dev, 8ull * ((uint64_t)F + 1), cudaMemcpyDeviceToHost, s));
    if (p->H) CK(cudaMemcpyAsync(o + L.holders, p->holders_dev, 12ull * p->H, cudaMemcpyDeviceToHost, s));
    unsigned long long hs[6] = {};
    CK(cudaMemcpyAsync(hs, ds, sizeof(hs), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    // host-side sections (capacities, bounds, class lists: the lists are gathered per worker
    // on the host copy) are summed with the same function
    auto hsum = [](const void* src, uint64_t words, int sec) {
        const uint32_t* w = static_cast<const uint32_t*>(src);
        uint64_t acc = 0;
        for (uint64_t i = 0; i < words; ++i) acc += mix64(((uint64_t)sec << 56) + i * kGolden) ^ (uint64_t)w[i];
        return acc;
    };
    h.checksum[0] = hsum(o + L.caps, 2ull * J, 0);
    h.checksum[1] = hs[1];
    h.checksum[2] = hsum(o + L.bounds, 4ull * nloc * J, 2);
    h.checksum[3] = hsum(o + L.lists, L.ncl, 3);
    h.checksum[4] = hs[4];
    h.checksum[5] = hs[5];
    memcpy(o, &h, sizeof(h));
    return 0;
}

int clairplan_wire_checksums(clairplan_t p, uint64_t stream_base, uint64_t list_base,
                             const uint64_t* d_holder_starts, uint64_t* out) {
    if (!p || !p->built || p->generic) return fail(CLAIRPLAN_EINVAL, "plan not built");
    if (!out) return fail(CLAIRPLAN_EINVAL, "null argument");
    CK(cudaSetDevice(p->device));
    cudaStream_t s = p->stream;
    const uint32_t J = p->cfg.num_classes, F = p->part.F;
    DevBuf sums;
    if (!sums.ensure(8 * 6)) return fail(CLAIRPLAN_ENOMEM, "device allocation failed");
    CK(cudaMemsetAsync(sums.p, 0, 8 * 6, s));
    unsigned long long* ds = sums.get<unsigned long long>();
    if (p->A)
        wire_sum_at_kernel<<<grid_for(p->A, kThreads, 148u * 8u), kThreads, 0, s>>>(
            p->stream_buf.get<uint32_t>(), p->A, stream_base, 1ull << 56, ds + 1);
    // class lists: (w, j) lists back to back, worker-major, from the list start of the shard
    uint64_t o = list_base;
    for (uint32_t w = 0; w < p->nloc; ++w)
        for (uint32_t j = 0; j < J; ++j) {
            const uint64_t n = p->class_len_h[(size_t)w * (J + 1) + j];
            const uint64_t st = p->class_start_h[(size_t)w * (J + 1) + j];
            if (n)
                wire_sum_at_kernel<<<grid_for(n, kThreads, 148u * 8u), kThreads, 0, s>>>(
                    p->class_entries.get<uint32_t>() + st, n, o, 3ull << 56, ds + 3);
            o += n;
        }
    if (!d_holder_starts) {
        wire_sum_kernel<<<grid_for(2 * ((uint64_t)F + 1), kThreads, 148u * 8u), kThreads, 0, s>>>(
            reinterpret_cast<const uint32_t*>(p->holder_off_dev), 2 * ((uint64_t)F + 1), 4ull << 56, ds + 4);
        if (p->H)
            wire_sum_kernel<<<grid_for(3 * p->H, kThreads, 148u * 8u), kThreads, 0, s>>>(
                p->holders_dev, 3 * p->H, 5ull << 56, ds + 5);
    } else if (p->H) {
        wire_holder_sum_kernel<<<grid_for(F, kThreads, 148u * 8u), kThreads, 0, s>>>(
            p->holders_dev, p->holder_off_dev, d_holder_starts, F, 5ull << 56, ds + 5);
    }
    CK(cudaGetLastError());
    unsigned long long hs[6] = {};
    CK(cudaMemcpyAsync(hs, ds, sizeof(hs), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    for (int i = 0; i < 6; ++i) out[i] = hs[i];
    return 0;
}

}  // extern "C"
