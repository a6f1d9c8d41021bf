// Plan consumer: the NoPFS source chooser over the holder CSR,
// batched on the device — one query per (sample, worker) access, e.g. every worker's batch of
// one simulator step (simulator.cpp:203-353 asks once per access).
//
//   choose_kernel   best_cached_source + choose_source (policies.cpp:168-233): walk the
//                   sample's holders (worker order); a holder is usable when the observing
//                   worker's prefetch progress in its class has passed its position
//                   (remote_available: the holder's own progress, or the requester's in
//                   heuristic mode); minimal unit fetch time, ties Local > Remote, then the
//                   lowest worker id; the cached source wins a tie against the PFS.
//   earliest_kernel the "earliest remote holder" table of the north star: per sample the
//                   holder with the smallest (remote unit fetch time, prefetch position,
//                   worker) — the copy a remote reader can expect first.  A derived view:
//                   the reference keeps no such table (it scans holders_of per access).
// Unit fetch times come from the caller's SystemConfig (fetch_time_local / _remote / _pfs at
// size 1.0, perfmodel.cpp:109-121): the comparisons are the reference's, on the same doubles.
#include "plan_impl.h"

namespace clairplan {

__global__ void choose_kernel(uint64_t n, const uint32_t* __restrict__ samples,
                              const uint32_t* __restrict__ workers,
                              const uint64_t* __restrict__ hoff, const uint32_t* __restrict__ hold,
                              const uint64_t* __restrict__ progress, uint32_t J,
                              const double* __restrict__ tl, const double* __restrict__ tr,
                              double tpfs, int allow_local, int allow_remote, int heuristic,
                              clairplan_source* __restrict__ out) {
    for (uint64_t x = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; x < n;
         x += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t s = samples[x], w = workers[x];
        double bt = 0;
        int brank = 2;
        uint32_t bw = kNone, bc = 0;
        bool found = false;
        for (uint64_t h = hoff[s], he = hoff[s + 1]; h < he; ++h) {
            const uint32_t hw = hold[3 * h], hc = hold[3 * h + 1], hpos = hold[3 * h + 2];
            int rank;
            double t;
            if (hw == w) {
                if (!allow_local || progress[(uint64_t)w * J + hc - 1] <= hpos) continue;
                rank = 0;
                t = tl[hc - 1];
            } else {
                const uint32_t obs = heuristic ? w : hw;
                if (!allow_remote || progress[(uint64_t)obs * J + hc - 1] <= hpos) continue;
                rank = 1;
                t = tr[hc - 1];
            }
            if (!found || t < bt || (t == bt && (rank < brank || (rank == brank && hw < bw)))) {
                found = true;
                bt = t;
                brank = rank;
                bw = hw;
                bc = hc;
            }
        }
        clairplan_source r{};
        if (found && bt <= tpfs) {
            r.kind = brank == 0 ? CLAIRPLAN_SRC_LOCAL : CLAIRPLAN_SRC_REMOTE;
            r.worker = brank == 0 ? w : bw;
            r.storage_class = (uint8_t)bc;
        } else {
            r.kind = CLAIRPLAN_SRC_PFS;
        }
        out[x] = r;
    }
}

__global__ void earliest_kernel(uint32_t F, const uint64_t* __restrict__ hoff,
                                const uint32_t* __restrict__ hold, const double* __restrict__ tr,
                                uint32_t* __restrict__ out) {
    for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < F; k += gridDim.x * blockDim.x) {
        uint32_t bw = kNone, bc = 0, bp = kNone;
        double bt = 0;
        for (uint64_t h = hoff[k], he = hoff[k + 1]; h < he; ++h) {
            const uint32_t hw = hold[3 * h], hc = hold[3 * h + 1], hp = hold[3 * h + 2];
            const double t = tr[hc - 1];
            if (bw == kNone || t < bt || (t == bt && (hp < bp || (hp == bp && hw < bw)))) {
                bw = hw;
                bc = hc;
                bp = hp;
                bt = t;
            }
        }
        out[3 * (uint64_t)k] = bw;
        out[3 * (uint64_t)k + 1] = bw == kNone ? kNone : bc;
        out[3 * (uint64_t)k + 2] = bp;
    }
}

}  // namespace clairplan

extern "C" {

int clairplan_choose_sources(clairplan_t p, uint64_t n, const uint32_t* samples,
                             const uint32_t* workers, const uint64_t* progress,
                             const double* local_time, const double* remote_time, double pfs_time,
                             int allow_local, int allow_remote, int heuristic, int on_device,
                             clairplan_source* out) {
    if (!p || !p->built) return fail(CLAIRPLAN_EINVAL, "plan not built");
    if (n && (!samples || !workers || !out)) return fail(CLAIRPLAN_EINVAL, "null argument");
    const uint32_t J = p->cfg.num_classes, N = p->part.N, F = p->part.F;
    if (J && (!progress || !local_time || !remote_time)) return fail(CLAIRPLAN_EINVAL, "null argument");
    if (n == 0) return 0;
    CK(cudaSetDevice(p->device));
    cudaStream_t s = p->stream;
    DevBuf q, prog, times, res;
    const uint32_t *ds = samples, *dw = workers;
    const uint64_t* dp = progress;
    clairplan_source* dout = out;
    if (!on_device) {
        if (!q.ensure(n * 8) || !prog.ensure(std::max<uint64_t>((uint64_t)N * J, 1) * 8) ||
            !res.ensure(n * sizeof(clairplan_source)))
            return fail(CLAIRPLAN_ENOMEM, "device allocation failed (source queries)");
        // the chooser reads samples / workers / progress as given: validate on the host
        for (uint64_t x = 0; x < n; ++x)
            if (samples[x] >= F || workers[x] >= N) return fail(CLAIRPLAN_EINVAL, "query out of range");
        CK(cudaMemcpyAsync(q.get<uint32_t>(), samples, n * 4, cudaMemcpyHostToDevice, s));
        CK(cudaMemcpyAsync(q.get<uint32_t>() + n, workers, n * 4, cudaMemcpyHostToDevice, s));
        if (J) CK(cudaMemcpyAsync(prog.p, progress, (uint64_t)N * J * 8, cudaMemcpyHostToDevice, s));
        ds = q.get<uint32_t>();
        dw = ds + n;
        dp = prog.get<uint64_t>();
        dout = res.get<clairplan_source>();
    }
    if (!times.ensure(std::max<uint32_t>(2 * J, 1) * 8)) return fail(CLAIRPLAN_ENOMEM, "device allocation failed");
    if (J) {
        CK(cudaMemcpyAsync(times.get<double>(), local_time, J * 8, cudaMemcpyHostToDevice, s));
        CK(cudaMemcpyAsync(times.get<double>() + J, remote_time, J * 8, cudaMemcpyHostToDevice, s));
    }
    if (p->H == 0 || !p->holders_dev) {
        // no holders: every access goes to the PFS
        std::vector<clairplan_source> pfs(n);
        for (auto& r : pfs) r = clairplan_source{CLAIRPLAN_SRC_PFS, 0, 0, 0};
        if (on_device) CK(cudaMemcpyAsync(out, pfs.data(), n * sizeof(clairplan_source), cudaMemcpyHostToDevice, s));
        else memcpy(out, pfs.data(), n * sizeof(clairplan_source));
        CK(cudaStreamSynchronize(s));
        return 0;
    }
    choose_kernel<<<grid_for(n, kThreads), kThreads, 0, s>>>(
        n, ds, dw, p->holder_off_dev, p->holders_dev, dp, J, times.get<double>(),
        times.get<double>() + J, pfs_time, allow_local, allow_remote, heuristic, dout);
    CK(cudaGetLastError());
    if (!on_device)
        CK(cudaMemcpyAsync(out, dout, n * sizeof(clairplan_source), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    return 0;
}

int clairplan_earliest_holders(clairplan_t p, const double* remote_time, uint32_t* out) {
    if (!p || !p->built) return fail(CLAIRPLAN_EINVAL, "plan not built");
    const uint32_t J = p->cfg.num_classes, F = p->part.F;
    if (!out || (J && !remote_time)) return fail(CLAIRPLAN_EINVAL, "null argument");
    CK(cudaSetDevice(p->device));
    cudaStream_t s = p->stream;
    DevBuf t, res;
    if (!res.ensure((uint64_t)F * 12) || !t.ensure(std::max<uint32_t>(J, 1) * 8))
        return fail(CLAIRPLAN_ENOMEM, "device allocation failed (earliest holders)");
    if (p->H == 0 || !p->holders_dev) {
        CK(cudaMemsetAsync(res.p, 0xFF, (uint64_t)F * 12, s));
    } else {
        CK(cudaMemcpyAsync(t.p, remote_time, J * 8, cudaMemcpyHostToDevice, s));
        earliest_kernel<<<grid_for(F, kThreads), kThreads, 0, s>>>(F, p->holder_off_dev, p->holders_dev,
                                                                   t.get<double>(), res.get<uint32_t>());
        CK(cudaGetLastError());
    }
    CK(cudaMemcpyAsync(out, res.p, (uint64_t)F * 12, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    return 0;
}

}  // extern "C"
