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

// Position-major: thread per permutation position p of the handle's workers in epochs
// [e_lo, e_hi) (epoch-major, so the inv rows being written stay L2-resident and their sectors
// are completed there): k = the stream entry at p, inv[e][k] = p.  Positions of the handle's
// workers in a full batch are contiguous: [h*B + sb(wb), h*B + sb(we)).
__global__ void __launch_bounds__(kThreads) stream_inv_kernel(Part part, uint32_t e_lo, uint32_t e_hi,
                                                              uint32_t lb, FastDiv dlb, uint32_t lt,
                                                              const uint32_t* __restrict__ stream,
                                                              uint32_t* __restrict__ inv) {
    const uint32_t F = part.F;
    const uint32_t sb = (uint32_t)(part.wbegin * part.base + min((uint64_t)part.wbegin, part.extra));
    const uint32_t tsb = (uint32_t)(part.wbegin * part.tbase + min((uint64_t)part.wbegin, part.textra));
    const uint64_t lfull = (uint64_t)part.full * lb;
    const uint64_t lep = lfull + lt;  // positions per epoch
    const uint64_t total = lep * (e_hi - e_lo);
    for (uint64_t x = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; x < total;
         x += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t el = (uint32_t)(x / lep);
        const uint32_t xe = (uint32_t)(x - (uint64_t)el * lep);
        const uint32_t e = e_lo + el;
        uint32_t pos;
        if (xe < lfull) {
            const uint32_t h = dlb.div(xe);
            pos = h * part.B + sb + (xe - h * lb);
        } else {
            pos = (uint32_t)(part.full * part.B) + tsb + (uint32_t)(xe - lfull);
        }
        uint32_t w;
        uint64_t spos;
        part.locate(pos, e, w, spos);
        const uint32_t k = __ldcs(stream + part.stream_offset(w) + spos);
        inv[(size_t)e * pitch16(F) + k] = pos;
    }
}

void launch_stream_relayout(cudaStream_t s, const Part& part, const EpochSplit& es,
                            const uint32_t* recv, uint32_t* stream) {
    const uint32_t nloc = part.wend - part.wbegin;
    dim3 grid(nloc * es.G, std::max<uint32_t>(1, (148u * 8u) / std::max<uint32_t>(1, nloc * es.G)));
    stream_relayout_kernel<<<grid, kThreads, 0, s>>>(part, es, recv, stream);
}

void launch_stream_inv(cudaStream_t s, const Part& part, const uint32_t* stream, uint32_t* inv,
                       uint32_t skip_lo, uint32_t skip_hi) {
    // epoch batches of ~40 MB of inv rows: the none-fill and the scatter of a batch meet in L2
    const uint32_t F = part.F, E = part.E;
    // local positions per full batch / in the tail batch
    const uint32_t lfb = (uint32_t)((part.wend * part.base + std::min<uint64_t>(part.wend, part.extra)) -
                                    (part.wbegin * part.base + std::min<uint64_t>(part.wbegin, part.extra)));
    const uint32_t ltb = part.tail ? (uint32_t)((part.wend * part.tbase + std::min<uint64_t>(part.wend, part.textra)) -
                                                (part.wbegin * part.tbase + std::min<uint64_t>(part.wbegin, part.textra)))
                                   : 0u;
    const uint32_t eb = std::max<uint32_t>(1, (uint32_t)((40ull << 20) / ((uint64_t)F * 4)));
    // epochs [skip_lo, skip_hi) already hold their whole inverse rows (the rank's own epochs,
    // written by clairplan_generate_streams): rebuilt are the others only
    for (uint32_t e0 = 0; e0 < E;) {
        if (e0 >= skip_lo && e0 < skip_hi) {
            e0 = skip_hi;
            continue;
        }
        const uint32_t e1 = std::min(std::min(E, e0 + eb), e0 < skip_lo ? skip_lo : E);
        cudaMemsetAsync(inv + (size_t)e0 * part.Fp, 0xFF, (size_t)(e1 - e0) * part.Fp * 4, s);
        const uint64_t n = ((uint64_t)part.full * lfb + ltb) * (e1 - e0);
        stream_inv_kernel<<<grid_for(n, kThreads, 148u * 16u), kThreads, 0, s>>>(
            part, e0, e1, lfb, FastDiv(lfb ? lfb : 1), ltb, stream, inv);
        e0 = e1;
    }
}

}  // namespace clairplan

// ---- holder-offset merge of a worker-sharded plan (DESIGN §6 step 4) -------------------
// allc[r][k] = holder records of sample k on rank r; the global CSR offset of k is the
// exclusive scan of the per-sample totals, and rank `rank`'s records of k start after those
// of ranks < rank (contiguous ascending worker ranges: build_index's worker order,
// policies.cpp:124-142).
namespace clairplan {

__global__ void merge_counts_kernel(const uint32_t* __restrict__ allc, uint32_t world, uint32_t rank,
                                    uint32_t F, uint32_t* __restrict__ tot, uint32_t* __restrict__ before) {
    for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < F; k += gridDim.x * blockDim.x) {
        uint32_t t = 0, b = 0;
        for (uint32_t r = 0; r < world; ++r) {
            const uint32_t c = allc[(uint64_t)r * F + k];
            t += c;
            b += r < rank ? c : 0u;
        }
        tot[k] = t;
        before[k] = b;
    }
}

__global__ void merge_starts_kernel(const uint64_t* __restrict__ glob, const uint32_t* __restrict__ before,
                                    uint32_t F, uint64_t* __restrict__ starts) {
    for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < F; k += gridDim.x * blockDim.x)
        starts[k] = glob[k] + before[k];
}

}  // namespace clairplan

#include "plan_impl.h"

extern "C" int clairplan_merge_holder_counts(clairplan_t p, const uint32_t* d_allc, uint32_t world,
                                             uint32_t rank, int64_t* d_glob, int64_t* d_starts,
                                             void* stream) {
    if (!p || !d_allc || !d_glob || !d_starts) return fail(CLAIRPLAN_EINVAL, "null argument");
    if (world < 1 || rank >= world) return fail(CLAIRPLAN_EINVAL, "invalid rank");
    CK(cudaSetDevice(p->device));
    const uint32_t F = p->part.F;
    // the caller's stream as given: 0 is the legacy default stream (torch's default stream,
    // where the all-gather of the counts ran), not "the handle's stream"
    cudaStream_t s = (cudaStream_t)stream;
    // own scratch: this may run while the handle's build is still in flight on p->stream
    // scan scratch: two (tiles + 1) u64 arrays per level, 256-B rounded (generous: a scratch
    // request that does not fit would hand the scan kernels a null pointer)
    const uint64_t nb = (uint64_t)F / 256 + 64;
    if (!p->merge_buf.ensure((uint64_t)F * 8 + 4 * nb * 8 + (64u << 10)))
        return fail(CLAIRPLAN_ENOMEM, "device allocation failed (holder merge)");
    uint32_t* tot = p->merge_buf.get<uint32_t>();
    uint32_t* before = tot + F;
    Workspace ws;
    ws.base = reinterpret_cast<char*>(p->merge_buf.get<uint32_t>() + 2 * (uint64_t)F);
    ws.base = reinterpret_cast<char*>(((uintptr_t)ws.base + 255) & ~(uintptr_t)255);
    ws.cap = p->merge_buf.bytes - (ws.base - p->merge_buf.get<char>());
    merge_counts_kernel<<<grid_for(F, kThreads), kThreads, 0, s>>>(d_allc, world, rank, F, tot, before);
    exclusive_scan(s, tot, F, reinterpret_cast<uint64_t*>(d_glob), ws);
    merge_starts_kernel<<<grid_for(F, kThreads), kThreads, 0, s>>>(reinterpret_cast<uint64_t*>(d_glob),
                                                                   before, F,
                                                                   reinterpret_cast<uint64_t*>(d_starts));
    CK(cudaGetLastError());
    if (ws.overflow) return fail(CLAIRPLAN_ENOMEM, "internal workspace overflow (holder merge)");
    return 0;
}
