// Entry points of the same path that do not start from the seed:
//   clairplan_access_frequencies    access_frequencies     (access.cpp:80-88)
//   clairplan_worker_access_counts  worker_access_counts   (access.cpp:90-102)
//   clairplan_all_access_counts     all_access_counts      (access.cpp:104-116)
//   clairplan_assign_from_streams   nopfs_assign_caches on caller streams + frequency tables
//                                   (policies.cpp:144-166, build_index :124-142)
//   clairplan_generate_sizes        DatasetModel::generate (perfmodel.cpp:68-99), host input
//
// nopfs_assign_caches takes arbitrary tables: candidates are the samples with counts > 0,
// ordered by (count desc, first stream position asc) where samples absent from the stream
// have first position kNoIndex (policies.cpp:12,16-23) and keep index order (stable_sort).
// So a worker's candidate list = [its first occurrences in stream order that have count>0]
// followed by [count>0 samples never read, ascending] — both stable compactions — and the
// rest of the pipeline (radix tier order, first fit, class lists) is shared with the seed
// path.  Holders are built by a stable radix sort of the assigned pairs on the sample id.
#include <math.h>

#include <cmath>

#include "plan_impl.h"

namespace clairplan {

__global__ void histogram_kernel(const uint32_t* __restrict__ entries, uint64_t n, uint32_t F,
                                 uint32_t* __restrict__ counts) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t k = entries[i];
        if (k < F) atomicAdd(&counts[k], 1u);
    }
}

// first stream position of every (w, k): dfirst[w*F + k]
__global__ void first_pos_kernel(const uint32_t* __restrict__ entries,
                                 const uint64_t* __restrict__ offs, uint32_t N, uint32_t F,
                                 uint32_t* __restrict__ dfirst) {
    for (uint32_t w = blockIdx.x; w < N; w += gridDim.x) {
        const uint64_t b = offs[w], L = offs[w + 1] - b;
        for (uint64_t i = threadIdx.x; i < L; i += blockDim.x)
            atomicMin(&dfirst[(uint64_t)w * F + entries[b + i]], (uint32_t)i);
    }
}

// key 0 = candidate, 1 = not, for the stream-order part (segments = worker streams)
__global__ void stream_cand_keys_kernel(const uint32_t* __restrict__ entries,
                                        const uint64_t* __restrict__ offs, uint32_t N, uint32_t F,
                                        const uint32_t* __restrict__ dfirst,
                                        const uint32_t* __restrict__ dcounts,
                                        uint32_t* __restrict__ keys) {
    for (uint32_t w = blockIdx.x; w < N; w += gridDim.x) {
        const uint64_t b = offs[w], L = offs[w + 1] - b;
        for (uint64_t i = threadIdx.x; i < L; i += blockDim.x) {
            const uint64_t x = (uint64_t)w * F + entries[b + i];
            keys[b + i] = (dfirst[x] == (uint32_t)i && dcounts[x] > 0) ? 0u : 1u;
        }
    }
}

// key 0 = count > 0 but never read (kNoIndex first position), over the dense [N][F] table
__global__ void unread_cand_keys_kernel(uint64_t NF, const uint32_t* __restrict__ dfirst,
                                        const uint32_t* __restrict__ dcounts,
                                        uint32_t* __restrict__ keys) {
    for (uint64_t x = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; x < NF;
         x += (uint64_t)gridDim.x * blockDim.x)
        keys[x] = (dfirst[x] == kNone && dcounts[x] > 0) ? 0u : 1u;
}

// candidates of worker w: n1 stream firsts (ovals1 = entry index) then n2 unread (ovals2 = w*F+k)
__global__ void gather_generic_cands_kernel(
    uint32_t N, uint32_t F, const uint32_t* __restrict__ entries,
    const uint64_t* __restrict__ r1s, const uint64_t* __restrict__ r1l,
    const uint32_t* __restrict__ v1, const uint64_t* __restrict__ r2s,
    const uint64_t* __restrict__ r2l, const uint32_t* __restrict__ v2,
    const uint64_t* __restrict__ cbase, const uint32_t* __restrict__ dcounts,
    uint32_t* __restrict__ cand_k, uint32_t* __restrict__ cand_cnt, uint32_t* __restrict__ cand_w,
    uint64_t* __restrict__ wbeg, uint64_t* __restrict__ wlen) {
    for (uint32_t w = blockIdx.x; w < N; w += gridDim.x) {
        const uint64_t o = cbase[w];
        const uint64_t n1 = r1l[w], n2 = r2l[w];
        if (threadIdx.x == 0) {
            wbeg[w] = o;
            wlen[w] = n1 + n2;
        }
        for (uint64_t i = threadIdx.x; i < n1; i += blockDim.x) {
            const uint32_t k = entries[v1[r1s[w] + i]];
            cand_k[o + i] = k;
            cand_cnt[o + i] = dcounts[(uint64_t)w * F + k];
            cand_w[o + i] = w;
        }
        for (uint64_t i = threadIdx.x; i < n2; i += blockDim.x) {
            const uint64_t x = v2[r2s[w] + i];  // dense index w*F + k
            const uint32_t k = (uint32_t)(x - (uint64_t)w * F);
            cand_k[o + n1 + i] = k;
            cand_cnt[o + n1 + i] = dcounts[x];
            cand_w[o + n1 + i] = w;
        }
    }
}

__global__ void sum_lens_kernel(const uint64_t* __restrict__ a, const uint64_t* __restrict__ b,
                                uint32_t n, uint64_t* __restrict__ out) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        out[i] = a[i] + b[i];
}

__global__ void generic_count_keys_kernel(const uint32_t* __restrict__ cnt, uint64_t n,
                                          uint32_t maxc, uint32_t* __restrict__ keys) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x)
        keys[i] = maxc - cnt[i];
}

void launch_generic_count_keys(cudaStream_t s, const uint32_t* cnt, uint64_t n, uint32_t maxc,
                               uint32_t* keys) {
    generic_count_keys_kernel<<<grid_for(n, kThreads), kThreads, 0, s>>>(cnt, n, maxc, keys);
}

// key = sample id of assigned pairs, F for unassigned (sorted last)
__global__ void holder_keys_kernel(const uint32_t* __restrict__ cand_k,
                                   const uint8_t* __restrict__ cand_cls, uint64_t n, uint32_t F,
                                   uint32_t* __restrict__ keys, uint32_t* __restrict__ hcount) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const bool a = cand_cls[i] != 0;
        keys[i] = a ? cand_k[i] : F;
        if (a) atomicAdd(&hcount[cand_k[i]], 1u);
    }
}

__global__ void holder_records_kernel(const uint32_t* __restrict__ sorted_idx, uint64_t H,
                                      const uint32_t* __restrict__ cand_w,
                                      const uint8_t* __restrict__ cand_cls,
                                      const uint32_t* __restrict__ dest,
                                      const uint64_t* __restrict__ class_start, uint32_t J,
                                      uint32_t* __restrict__ holders) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < H;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t c = sorted_idx[i];
        const uint32_t w = cand_w[c], cls = cand_cls[c];
        holders[3 * i + 0] = w;
        holders[3 * i + 1] = cls;
        holders[3 * i + 2] = (uint32_t)(dest[c] - class_start[(uint64_t)w * (J + 1) + cls - 1]);
    }
}

int generic_holders(clairplan_plan* p) {
    cudaStream_t s = p->stream;
    const uint64_t D = p->D;
    const uint32_t F = p->part.F, J = p->cfg.num_classes, N = p->nloc;
    CK(cudaStreamSynchronize(s));
    uint64_t H = 0;
    for (uint32_t w = 0; w < N; ++w)
        for (uint32_t d = 0; d < J; ++d) H += p->class_len_h[(size_t)w * (J + 1) + d];
    p->H = H;
    bool ok = true;
    uint32_t* hc = need<uint32_t>(p->hcount, F, ok);
    uint64_t* ho = need<uint64_t>(p->hoff, (uint64_t)F + 1, ok);
    uint32_t* hl = need<uint32_t>(p->holders, 3 * std::max<uint64_t>(H, 1), ok);
    if (!ok) return fail(CLAIRPLAN_ENOMEM, "device allocation failed (holders)");
    Workspace& ws = p->ws;
    ws.used = 0;
    CK(cudaMemsetAsync(hc, 0, (size_t)F * 4, s));
    uint32_t* keys = p->keys.get<uint32_t>();
    uint32_t* okeys = p->okeys.get<uint32_t>();
    uint32_t* vals = p->vals.get<uint32_t>();
    uint32_t* ovals = p->ovals.get<uint32_t>();
    holder_keys_kernel<<<grid_for(D, kThreads), kThreads, 0, s>>>(
        p->cand_k.get<uint32_t>(), p->cand_cls.get<uint8_t>(), D, F, keys, hc);
    exclusive_scan(s, hc, F, ho, ws);
    // one segment over all candidates: stable sort on the sample id (worker order kept)
    uint64_t* seg = ws.scratch<uint64_t>(2);
    const uint64_t hseg[2] = {0, D};
    CK(cudaMemcpyAsync(seg, hseg, 16, cudaMemcpyHostToDevice, s));
    TileMap tm;
    build_tilemap(s, seg + 1, 1, D, kRadixTile, tm, ws);
    const uint32_t* kin = keys;
    const uint32_t* vin = nullptr;
    uint32_t pass = 0;
    for (uint32_t shift = 0; shift == 0 || ((uint64_t)F >> shift) != 0; shift += 8, ++pass) {
        uint32_t* ko = (pass & 1) ? keys : okeys;
        uint32_t* vo = (pass & 1) ? vals : ovals;
        const size_t m = ws.mark();
        radix_pass(s, tm, seg, seg + 1, kin, vin, shift, ko, vo, nullptr, nullptr, ws);
        ws.release(m);
        kin = ko;
        vin = vo;
    }
    if (H)
        holder_records_kernel<<<grid_for(H, kThreads), kThreads, 0, s>>>(
            vin, H, p->cand_w.get<uint32_t>(), p->cand_cls.get<uint8_t>(), p->dest.get<uint32_t>(),
            p->class_start.get<uint64_t>(), J, hl);
    CK(cudaStreamSynchronize(s));
    CK(cudaGetLastError());
    if (ws.overflow) return fail(CLAIRPLAN_ENOMEM, "internal workspace overflow");
    p->holder_off_dev = ho;
    p->holders_dev = hl;
    return 0;
}


// ---- build_index (policies.cpp:124-142) on caller class lists ---------------------------
// entries: all class lists concatenated in (worker, class) order; list_off[N*J + 1].
__global__ void index_records_kernel(const uint64_t* __restrict__ list_off, uint32_t nlists,
                                     uint32_t J, uint64_t n, uint32_t* __restrict__ wj,
                                     uint32_t* __restrict__ pos) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t lo = 0, hi = nlists;  // last list with list_off[x] <= i
        while (hi - lo > 1) {
            const uint32_t mid = (lo + hi) / 2;
            if (list_off[mid] <= i) lo = mid;
            else hi = mid;
        }
        wj[i] = lo;
        pos[i] = (uint32_t)(i - list_off[lo]);
    }
}

__global__ void index_emit_kernel(const uint32_t* __restrict__ sorted_idx, uint64_t n,
                                  const uint32_t* __restrict__ wj, const uint32_t* __restrict__ pos,
                                  uint32_t J, uint32_t* __restrict__ holders) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t x = sorted_idx[i];
        holders[3 * i + 0] = wj[x] / J;
        holders[3 * i + 1] = wj[x] % J + 1;
        holders[3 * i + 2] = pos[x];
    }
}

}  // namespace clairplan
using namespace clairplan;
extern "C" int clairplan_build_index(uint32_t N, uint32_t J, uint64_t samples,
                                     const uint32_t* entries, const uint64_t* list_off,
                                     uint64_t* offsets_out, uint32_t* holders_out, int device) {
    if (!list_off || !offsets_out) return fail(CLAIRPLAN_EINVAL, "null argument");
    if (samples >= 0xFFFFFFFFull) return fail(CLAIRPLAN_EOVERFLOW, "too many samples");
    const uint32_t nl = N * J;
    const uint64_t n = nl ? list_off[nl] : 0;
    for (uint64_t i = 0; i < n; ++i)
        if (entries[i] >= samples) return fail(CLAIRPLAN_EINVAL, "class list entry out of range");
    if (int rc = check_device(device)) return rc;
    const uint32_t F = (uint32_t)samples;
    cudaStream_t s;
    CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    DevBuf dent, doff, dwj, dpos, keys, okeys, vals, ovals, hc, ho, hold, wsb;
    const uint64_t m = n ? n : 1;
    if (!dent.ensure(m * 4) || !doff.ensure(((uint64_t)nl + 1) * 8) || !dwj.ensure(m * 4) ||
        !dpos.ensure(m * 4) || !keys.ensure(m * 4) || !okeys.ensure(m * 4) || !vals.ensure(m * 4) ||
        !ovals.ensure(m * 4) || !hc.ensure(((uint64_t)F + 1) * 4) || !ho.ensure(((uint64_t)F + 1) * 8) ||
        !hold.ensure(m * 12)) {
        cudaStreamDestroy(s);
        return fail(CLAIRPLAN_ENOMEM, "device allocation failed");
    }
    const uint64_t ws_bytes = 256ull * (n / kRadixTile + 3) * 12 * 2 + (64ull << 20);
    if (!wsb.ensure(ws_bytes)) {
        cudaStreamDestroy(s);
        return fail(CLAIRPLAN_ENOMEM, "device allocation failed");
    }
    Workspace ws;
    ws.base = wsb.get<char>();
    ws.cap = wsb.bytes;
    CK(cudaMemsetAsync(hc.p, 0, ((uint64_t)F + 1) * 4, s));
    if (n) {
        CK(cudaMemcpyAsync(dent.p, entries, n * 4, cudaMemcpyHostToDevice, s));
        CK(cudaMemcpyAsync(doff.p, list_off, ((uint64_t)nl + 1) * 8, cudaMemcpyHostToDevice, s));
        CK(cudaMemcpyAsync(keys.p, entries, n * 4, cudaMemcpyHostToDevice, s));
        histogram_kernel<<<grid_for(n, kThreads), kThreads, 0, s>>>(dent.get<uint32_t>(), n, F,
                                                                   hc.get<uint32_t>());
        index_records_kernel<<<grid_for(n, kThreads), kThreads, 0, s>>>(
            doff.get<uint64_t>(), nl, J, n, dwj.get<uint32_t>(), dpos.get<uint32_t>());
    }
    exclusive_scan(s, hc.get<uint32_t>(), F, ho.get<uint64_t>(), ws);
    if (n) {
        uint64_t* seg = ws.scratch<uint64_t>(2);
        const uint64_t hseg[2] = {0, n};
        CK(cudaMemcpyAsync(seg, hseg, 16, cudaMemcpyHostToDevice, s));
        TileMap tm;
        build_tilemap(s, seg + 1, 1, n, kRadixTile, tm, ws);
        const uint32_t* kin = keys.get<uint32_t>();
        const uint32_t* vin = nullptr;
        uint32_t pass = 0;
        for (uint32_t shift = 0; shift == 0 || ((uint64_t)(F - 1) >> shift) != 0; shift += 8, ++pass) {
            uint32_t* ko = (pass & 1) ? keys.get<uint32_t>() : okeys.get<uint32_t>();
            uint32_t* vo = (pass & 1) ? vals.get<uint32_t>() : ovals.get<uint32_t>();
            const size_t mk = ws.mark();
            radix_pass(s, tm, seg, seg + 1, kin, vin, shift, ko, vo, nullptr, nullptr, ws);
            ws.release(mk);
            kin = ko;
            vin = vo;
        }
        index_emit_kernel<<<grid_for(n, kThreads), kThreads, 0, s>>>(vin, n, dwj.get<uint32_t>(),
                                                                    dpos.get<uint32_t>(), J,
                                                                    hold.get<uint32_t>());
    }
    CK(cudaMemcpyAsync(offsets_out, ho.p, ((uint64_t)F + 1) * 8, cudaMemcpyDeviceToHost, s));
    if (n) CK(cudaMemcpyAsync(holders_out, hold.p, n * 12, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    CK(cudaGetLastError());
    cudaStreamDestroy(s);
    if (ws.overflow) return fail(CLAIRPLAN_ENOMEM, "internal workspace overflow");
    return 0;
}
namespace clairplan {
}  // namespace clairplan

using namespace clairplan;

extern "C" {

int clairplan_access_frequencies(const uint32_t* entries, const uint64_t* epoch_offsets,
                                 uint32_t epoch_count, uint32_t samples, uint32_t eb, uint32_t ee,
                                 uint32_t* counts, int device) {
    if (int rc = check_device(device)) return rc;
    if (ee > epoch_count) ee = epoch_count;  // access.cpp:85 (e < stream.epoch_count())
    const uint64_t a = eb < ee ? epoch_offsets[eb] : 0, b = eb < ee ? epoch_offsets[ee] : 0;
    DevBuf de, dc;
    if (!dc.ensure((size_t)samples * 4 + 4) || !de.ensure((b - a) * 4 + 4))
        return fail(CLAIRPLAN_ENOMEM, "device allocation failed");
    CK(cudaMemset(dc.p, 0, (size_t)samples * 4));
    if (b > a) {
        CK(cudaMemcpy(de.p, entries + a, (b - a) * 4, cudaMemcpyHostToDevice));
        histogram_kernel<<<grid_for(b - a, kThreads), kThreads>>>(de.get<uint32_t>(), b - a, samples,
                                                                 dc.get<uint32_t>());
        CK(cudaGetLastError());
    }
    CK(cudaMemcpy(counts, dc.p, (size_t)samples * 4, cudaMemcpyDeviceToHost));
    return 0;
}

static int counts_plan(const clairplan_config* cfg, uint32_t wb, uint32_t we, clairplan_t* out) {
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

int clairplan_worker_access_counts(const clairplan_config* cfg, uint32_t worker, uint32_t* counts) {
    if (!cfg) return fail(CLAIRPLAN_EINVAL, "null config");
    if (int rc = clairplan_validate(cfg)) return rc;
    if (worker >= cfg->num_workers) return fail(CLAIRPLAN_EINVAL, "worker out of range");
    clairplan_t p = nullptr;
    if (int rc = counts_plan(cfg, worker, worker + 1, &p)) return rc;
    const int rc = clairplan_export_counts(p, worker, counts);
    clairplan_destroy(p);
    return rc;
}

int clairplan_all_access_counts(const clairplan_config* cfg, uint32_t* counts) {
    if (!cfg) return fail(CLAIRPLAN_EINVAL, "null config");
    if (int rc = clairplan_validate(cfg)) return rc;
    clairplan_t p = nullptr;
    if (int rc = counts_plan(cfg, 0, cfg->num_workers, &p)) return rc;
    for (uint32_t w = 0; w < cfg->num_workers; ++w) {
        if (int rc = clairplan_export_counts(p, w, counts + (uint64_t)w * cfg->samples)) {
            clairplan_destroy(p);
            return rc;
        }
    }
    clairplan_destroy(p);
    return 0;
}

int clairplan_assign_from_streams(uint32_t N, uint32_t F, const uint32_t* entries,
                                  const uint64_t* offsets, const uint32_t* counts, uint32_t J,
                                  const double* caps, const double* sizes, int device,
                                  clairplan_t* out) {
    if (!out || !offsets || !counts || (J && !caps) || !sizes)
        return fail(CLAIRPLAN_EINVAL, "null argument");
    *out = nullptr;
    if (N < 1 || F < 1) return fail(CLAIRPLAN_EINVAL, "num_workers and samples must be >= 1");
    if (J > 254) return fail(CLAIRPLAN_EINVAL, "device plan supports at most 254 cache classes");
    const uint64_t A = offsets[N];
    for (uint32_t w = 0; w < N; ++w)
        if (offsets[w + 1] - offsets[w] >= 0xFFFFFFFFull)
            return fail(CLAIRPLAN_EOVERFLOW, "stream longer than 2^32-1 entries");
    for (uint64_t i = 0; i < A; ++i)
        if (entries[i] >= F) return fail(CLAIRPLAN_EINVAL, "stream entry out of range");
    if ((uint64_t)N * F >= 0xFFFFFFFFull)
        return fail(CLAIRPLAN_EOVERFLOW, "N x F frequency table too large for one handle");
    if (int rc = check_device(device)) return rc;
    auto* p = new clairplan_plan();
    auto bail = [&](int rc) {
        delete p;
        return rc;
    };
    p->device = device;
    p->generic = true;
    p->cfg.samples = F;
    p->cfg.num_workers = N;
    p->cfg.num_classes = J;
    p->cfg.device = device;
    p->cfg.worker_begin = 0;
    p->cfg.worker_end = N;
    p->caps.assign(caps, caps + J);
    p->part = make_part(F, N, N, 1, true, 0, N);
    p->nloc = N;
    p->A = A;
    if (cudaStreamCreateWithFlags(&p->stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreate(&p->ev0) != cudaSuccess || cudaEventCreate(&p->ev1) != cudaSuccess)
        return bail(fail(CLAIRPLAN_ECUDA, "stream/event creation failed"));
    cudaStream_t s = p->stream;
    const uint64_t NF = (uint64_t)N * F;
    uint32_t maxc = 0;
    for (uint64_t x = 0; x < NF; ++x) maxc = counts[x] > maxc ? counts[x] : maxc;
    p->maxcount = maxc;
    bool ok = true;
    double* dsz = need<double>(p->sizes, F, ok);
    uint32_t* dent = need<uint32_t>(p->stream_buf, A, ok);
    uint32_t* dcnt = need<uint32_t>(p->dcounts, NF, ok);
    uint32_t* dfirst = need<uint32_t>(p->dfirst, NF, ok);
    uint64_t* doff = need<uint64_t>(p->seg_off, (uint64_t)N + 1, ok);
    uint64_t* dlen = need<uint64_t>(p->segcnt, (uint64_t)N * 8, ok);
    uint32_t* keys = need<uint32_t>(p->keys, std::max(A, NF), ok);
    uint32_t* okeys = need<uint32_t>(p->okeys, std::max(A, NF), ok);
    uint32_t* ov1 = need<uint32_t>(p->ovals, std::max(A, NF), ok);
    uint32_t* ov2 = need<uint32_t>(p->vals, std::max(A, NF), ok);
    if (!ok) return bail(fail(CLAIRPLAN_ENOMEM, "device allocation failed"));
    if (int rc = ensure_ws(p, std::max(A, NF), N)) return bail(rc);
    Workspace& ws = p->ws;
    CK(cudaMemcpyAsync(dsz, sizes, (size_t)F * 8, cudaMemcpyHostToDevice, s));
    if (A) CK(cudaMemcpyAsync(dent, entries, A * 4, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(dcnt, counts, NF * 4, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(doff, offsets, ((uint64_t)N + 1) * 8, cudaMemcpyHostToDevice, s));
    CK(cudaMemsetAsync(dfirst, 0xFF, NF * 4, s));
    first_pos_kernel<<<grid_for(N, 1, 148u * 16u), kThreads, 0, s>>>(dent, doff, N, F, dfirst);
    stream_cand_keys_kernel<<<grid_for(N, 1, 148u * 16u), kThreads, 0, s>>>(dent, doff, N, F,
                                                                            dfirst, dcnt, keys);
    // segment arrays: [0,N) stream begins, [N,2N) stream lens, [2N,3N) dense begins, [3N,4N) dense lens
    std::vector<uint64_t> hs(4 * (size_t)N);
    for (uint32_t w = 0; w < N; ++w) {
        hs[w] = offsets[w];
        hs[N + w] = offsets[w + 1] - offsets[w];
        hs[2 * N + w] = (uint64_t)w * F;
        hs[3 * N + w] = F;
    }
    CK(cudaMemcpyAsync(dlen, hs.data(), hs.size() * 8, cudaMemcpyHostToDevice, s));
    uint64_t* r = dlen + 4 * (uint64_t)N;  // regions: r1s, r1l, r2s, r2l
    {
        TileMap tm;
        const size_t m = ws.mark();
        build_tilemap(s, dlen + N, N, A, kRadixTile, tm, ws);
        uint64_t* sc = nullptr;
        radix_pass(s, tm, dlen, dlen + N, keys, nullptr, 0, okeys, ov1, nullptr, &sc, ws);
        radix_regions(s, tm, dlen, dlen + N, sc, 1, r, r + N);
        ws.release(m);
    }
    unread_cand_keys_kernel<<<grid_for(NF, kThreads), kThreads, 0, s>>>(NF, dfirst, dcnt, keys);
    {
        TileMap tm;
        const size_t m = ws.mark();
        build_tilemap(s, dlen + 3 * (uint64_t)N, N, NF, kRadixTile, tm, ws);
        uint64_t* sc = nullptr;
        // values default to the global dense index w*F + k
        radix_pass(s, tm, dlen + 2 * (uint64_t)N, dlen + 3 * (uint64_t)N, keys, nullptr, 0, okeys,
                   ov2, nullptr, &sc, ws);
        radix_regions(s, tm, dlen + 2 * (uint64_t)N, dlen + 3 * (uint64_t)N, sc, 1, r + 2 * N,
                      r + 3 * N);
        ws.release(m);
    }
    // candidate bases: exclusive scan of n1 + n2
    uint64_t* tot = ws.scratch<uint64_t>(N);
    uint64_t* cbase = ws.scratch<uint64_t>((uint64_t)N + 1);
    sum_lens_kernel<<<grid_for(N, kThreads), kThreads, 0, s>>>(r + N, r + 3 * (uint64_t)N, N, tot);
    exclusive_scan(s, tot, N, cbase, ws);
    uint64_t D = 0;
    CK(cudaMemcpyAsync(&D, cbase + N, 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (D >= 0xFFFFFFFFull) return bail(fail(CLAIRPLAN_EOVERFLOW, "too many candidates"));
    p->D = D;
    uint32_t* ck = need<uint32_t>(p->cand_k, D, ok);
    uint32_t* cc = need<uint32_t>(p->cand_info, D, ok);
    uint32_t* cw = need<uint32_t>(p->cand_w, D, ok);
    uint64_t* wbeg = need<uint64_t>(p->wbeg, N, ok);
    uint64_t* wlen = need<uint64_t>(p->wlen, N, ok);
    if (!ok) return bail(fail(CLAIRPLAN_ENOMEM, "device allocation failed (candidates)"));
    gather_generic_cands_kernel<<<grid_for(N, 1, 148u * 16u), kThreads, 0, s>>>(
        N, F, dent, r, r + N, ov1, r + 2 * (uint64_t)N, r + 3 * (uint64_t)N, ov2, cbase, dcnt, ck,
        cc, cw, wbeg, wlen);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(s));
    if (J > 0) {
        if (int rc = assign_tiers(p)) return bail(rc);
    } else {
        p->H = 0;
        uint64_t* ho = need<uint64_t>(p->hoff, (uint64_t)F + 1, ok);
        if (!ok) return bail(fail(CLAIRPLAN_ENOMEM, "device allocation failed"));
        CK(cudaMemsetAsync(ho, 0, ((uint64_t)F + 1) * 8, s));
        p->holder_off_dev = ho;
        p->class_start_h.assign(N, 0);
        p->class_len_h.assign(N, 0);
    }
    CK(cudaStreamSynchronize(s));
    p->built = true;
    *out = p;
    return 0;
}

// DatasetModel::generate (perfmodel.cpp:68-99) — host-side input.  CounterRng::normal is
// rng.cpp:7-13 (cosine branch of Box-Muller, glibc sqrt/log/cos).
int clairplan_generate_sizes(uint64_t F, double mean, double sigma_in, int has_total,
                             double total, uint64_t seed, int sigma_relative, double* out) {
    if (F < 1) return fail(CLAIRPLAN_EINVAL, "dataset must have at least one sample");
    if (mean <= 0) return fail(CLAIRPLAN_EINVAL, "mean size must be positive");
    if (sigma_in < 0) return fail(CLAIRPLAN_EINVAL, "sigma must be >= 0");
    const double sigma = sigma_relative ? sigma_in * mean : sigma_in;
    const double floor_mb = std::min(std::max(1e-3, mean / 100.0), mean);
    const uint64_t key = derive_key(seed, kSizeTag);
    uint64_t pos = 0;
    double sum = 0;
    for (uint64_t k = 0; k < F; ++k) {
        double v;
        if (sigma == 0) {
            v = mean;
        } else {
            const double u1 = (double)(mix64(key + (++pos) * kGolden) >> 11) * 0x1.0p-53;
            const double u2 = (double)(mix64(key + (++pos) * kGolden) >> 11) * 0x1.0p-53;
            const double rr = std::sqrt(-2.0 * std::log(1.0 - u1));
            const double z = rr * std::cos(2.0 * M_PI * u2);
            v = std::max(floor_mb, mean + sigma * z);
        }
        out[k] = v;
        sum += v;
    }
    if (has_total) {
        const double scale = total / sum;
        for (uint64_t k = 0; k < F; ++k) out[k] *= scale;
    }
    return 0;
}

}  // extern "C"
