// clairplan C ABI (include/clairplan.h): host orchestration of the device plan build.
//
// Pipeline of clairplan_build (one CUDA stream per handle, 2 host syncs):
//   K1-K3 fy_link / fy_group / fy_emit   per batch of epochs: permutation -> streams + inv
//   K4a   sample_pass                    per sample: (w,k) counts, first epoch, holder rank
//         scan(pair_count)               -> pair offsets (= holder_offsets when all assigned)
//   K4b   seg_count, scan, seg_write     -> candidates per worker in first-access order
//   K5    radix pass on (E - count)      -> tier order (count desc, first asc)
//   K6    first_fit_pass per class       -> class of every candidate
//   K7    radix pass on class digit      -> prefetch-ordered class lists
//   K8    holder_scatter (+ compaction)  -> holder CSR
#include <stdlib.h>
#include <cstring>

#include "plan_impl.h"

namespace clairplan {
thread_local std::string g_err;

}  // namespace clairplan

namespace clairplan {

uint32_t epochs_per_batch(uint32_t F, uint32_t E, uint32_t bytes_per_target) {
    const uint64_t per = (uint64_t)F * bytes_per_target;
    uint64_t budget = 4096ull << 20;  // B200: 180 GB HBM; whole-run batches fill the GPU
    budget = (uint64_t)ab_knob("CLAIRPLAN_PERM_BUDGET_MB", 4096) << 20;
    uint64_t eb = budget / (per ? per : 1);
    if (eb < 1) eb = 1;
    if (eb > E) eb = E;
    if (eb > 128) eb = 128;
    return (uint32_t)eb;
}

RejTable rej_table(clairplan_plan* p) {
    RejTable rt;
    rt.step = p->rej_step.get<uint32_t>();
    rt.cum = p->rej_cum.get<uint32_t>();
    rt.count = p->rej_count.get<uint32_t>();
    rt.cap = kRejCap;
    rt.e_base = p->rej_ebase;
    return rt;
}

// Geometry of the contiguous-bucket shuffle for F (computed once per handle, uploaded once).
bool fyc_ready(clairplan_plan* p, uint32_t F, FycDev& g) {
    if (p->fyc_off) return false;
    FycHost& h = p->fych;
    if (h.F != F) {
        if (!fyc_plan(F, h)) {
            h.F = 0;
            return false;
        }
        const uint64_t nb = h.NB + 1, nc = h.cell.size();
        if (!p->fyc_geo.ensure((3 * nb + nc) * 4)) {
            h.F = 0;
            return false;
        }
        std::vector<uint32_t> buf;
        buf.reserve(3 * nb + nc);
        buf.insert(buf.end(), h.bstart.begin(), h.bstart.end());
        buf.insert(buf.end(), h.cap.begin(), h.cap.end());
        buf.push_back(0);
        for (uint64_t x : h.roff) buf.push_back((uint32_t)x);
        buf.insert(buf.end(), h.cell.begin(), h.cell.end());
        // stream-ordered with the shuffle kernels (a plain cudaMemcpy from pageable memory may
        // return before its DMA lands, and the handle's stream does not wait for the legacy
        // stream); pageable source: the call returns once the buffer is staged
        if (cudaMemcpyAsync(p->fyc_geo.p, buf.data(), buf.size() * 4, cudaMemcpyHostToDevice,
                            p->stream) != cudaSuccess) {
            cudaGetLastError();
            h.F = 0;
            return false;
        }
    }
    const uint32_t* d = p->fyc_geo.get<uint32_t>();
    const uint64_t nb = h.NB + 1;
    g.NB = h.NB;
    g.lgW = h.lgW;
    g.pack = h.pack;
    g.rtotal = h.rtotal;
    g.bstart = d;
    g.cap = d + nb;
    g.roff = d + 2 * nb;
    g.cell = d + 3 * nb;
    return true;
}

// Enqueues the permutations of epochs [e_first, e_first + e_count): stream + inverse (or plain
// permutations).  `spart` (optional) replaces the handle's stream geometry.
int enqueue_perms(clairplan_plan* p, uint32_t* stream_out, uint32_t* inv_out, uint32_t* perm_out,
                  uint32_t e_first, uint32_t e_count, const Part* spart = nullptr,
                  const StreamDst* dst = nullptr) {
    const Part& part = spart ? *spart : p->part;  // stream geometry (epoch-range streams)
    const uint32_t F = part.F;
    bool ok = true;
    const RejTable rt = rej_table(p);
    // contiguous-bucket resolution; the linked-list one (perm.cu) after a bucket overflow or
    // where the geometry does not apply (CLAIRPLAN_FY_LISTS forces it: parity coverage)
    const bool lists = path_switch("CLAIRPLAN_FY_LISTS") != nullptr;
    FycDev fg;
    if (!lists && fyc_ready(p, F, fg)) {  // contiguous target-block buckets
        const uint32_t EB = fyc_epochs_per_batch(F, e_count);
        uint32_t* region = need<uint32_t>(p->fyc_region, (uint64_t)EB * fg.rtotal, ok);
        uint32_t* cursor = need<uint32_t>(p->fyc_cursor, (uint64_t)EB * fg.NB + 1, ok);  // + emit claim
        uint32_t* tsucc = need<uint32_t>(p->next, (uint64_t)EB * F, ok);
        uint32_t* q = need<uint32_t>(p->q, (uint64_t)EB * F, ok);
        if (!ok) return fail(CLAIRPLAN_ENOMEM, "device allocation failed (permutation workspace)");
        for (uint32_t e0 = e_first; e0 < e_first + e_count; e0 += EB) {
            const uint32_t ne = std::min(EB, e_first + e_count - e0);
            launch_fyc(p->stream, p->key, part, e0, ne, fg, rt, p->rej_flag.get<uint32_t>(), region,
                       cursor, tsucc, q, inv_out, stream_out,
                       perm_out ? perm_out + (size_t)(e0 - e_first) * F : nullptr, dst);
            p->launches += 4;
        }
        CK(cudaGetLastError());
        return 0;
    }
    if (dst && dst->G) return fail(CLAIRPLAN_EINVAL, "peer-memory stream writes need the bucketed shuffle");
    const uint32_t EB = epochs_per_batch(F, e_count, 12);
    uint32_t* head = need<uint32_t>(p->head, (uint64_t)EB * F, ok);
    uint32_t* next = need<uint32_t>(p->next, (uint64_t)EB * F, ok);
    uint32_t* q = need<uint32_t>(p->q, (uint64_t)EB * F, ok);
    const uint32_t scap = 1u << 20;
    uint32_t* scratch = need<uint32_t>(p->scratch, scap, ok);
    uint32_t* counters = need<uint32_t>(p->counters, 4, ok);
    if (!ok) return fail(CLAIRPLAN_ENOMEM, "device allocation failed (permutation workspace)");
    for (uint32_t e0 = e_first; e0 < e_first + e_count; e0 += EB) {
        const uint32_t ne = std::min(EB, e_first + e_count - e0);
        CK(cudaMemsetAsync(head, 0xFF, (size_t)ne * F * sizeof(uint32_t), p->stream));
        CK(cudaMemsetAsync(counters, 0, 2 * sizeof(uint32_t), p->stream));  // cursor + overflow
        launch_fy_link(p->stream, p->key, F, e0, ne, head, next, rt, p->rej_flag.get<uint32_t>(),
                       false, F);
        launch_fy_group(p->stream, F, ne, head, next, q, scratch, scap, counters, counters + 1);
        launch_fy_emit(p->stream, p->key, part, e0, ne, next, q, rt, inv_out, stream_out,
                       perm_out ? perm_out + (size_t)(e0 - e_first) * F : nullptr);
        p->launches += 3;
        // fy_group's long-list scratch overflowed (never seen: lists at target y are ~ln(F/y)
        // long): its targets were not linked, so refuse rather than return a wrong plan
        uint32_t ovf = 0;
        CK(cudaMemcpyAsync(&ovf, counters + 1, sizeof(uint32_t), cudaMemcpyDeviceToHost, p->stream));
        CK(cudaStreamSynchronize(p->stream));
        if (ovf) return fail(CLAIRPLAN_ENOMEM, "linked-list shuffle: long-list scratch overflow");
    }
    CK(cudaGetLastError());
    return 0;
}

// Resolves Lemire rejections (rng.hpp:54-60) of the flagged epochs into the per-epoch
// shift tables.  Rare: ~F^2/2^66 rejections per epoch.
int resolve_rejections(clairplan_plan* p, const std::vector<uint32_t>& flags, bool* any) {
    *any = false;
    const uint32_t F = p->part.F;
    for (uint32_t er = 0; er < flags.size(); ++er) {
        const uint32_t e = er + p->rej_ebase;
        uint32_t flag = flags[er];
        if (flag & kRejOverflow) {
            // a contiguous-bucket region overflowed (mean + 10 sigma exceeded): rerun the
            // shuffle on the linked-list path; its own detection finds any rejection again
            p->fyc_off = true;
            *any = true;
            CK(cudaMemsetAsync(p->rej_flag.get<uint32_t>() + er, 0, sizeof(uint32_t), p->stream));
            continue;
        }
        while (flag) {
            *any = true;
            const uint32_t i = flag - 1;
            uint32_t* st = &p->rej_step_h[(size_t)er * kRejCap];
            uint32_t* cu = &p->rej_cum_h[(size_t)er * kRejCap];
            uint32_t& n = p->rej_count_h[er];
            if (n >= kRejCap) return fail(CLAIRPLAN_EOVERFLOW, "too many Lemire rejections in one epoch");
            const uint32_t shift = rej_shift(st, cu, n, i);
            uint32_t extra = 0;
            fy_draw(p->key, e, F, i, shift, &extra);
            st[n] = i;
            cu[n] = shift + extra;
            ++n;
            ++p->rejections;
            CK(cudaMemcpyAsync(p->rej_step.get<uint32_t>() + (size_t)er * kRejCap, st,
                               kRejCap * sizeof(uint32_t), cudaMemcpyHostToDevice, p->stream));
            CK(cudaMemcpyAsync(p->rej_cum.get<uint32_t>() + (size_t)er * kRejCap, cu,
                               kRejCap * sizeof(uint32_t), cudaMemcpyHostToDevice, p->stream));
            CK(cudaMemcpyAsync(p->rej_count.get<uint32_t>() + er, &n, sizeof(uint32_t),
                               cudaMemcpyHostToDevice, p->stream));
            CK(cudaMemsetAsync(p->rej_flag.get<uint32_t>() + er, 0, sizeof(uint32_t), p->stream));
            launch_fy_link(p->stream, p->key, F, e, 1, nullptr, nullptr, rej_table(p),
                           p->rej_flag.get<uint32_t>(), true, i);
            ++p->launches;
            CK(cudaMemcpyAsync(&flag, p->rej_flag.get<uint32_t>() + er, sizeof(uint32_t),
                               cudaMemcpyDeviceToHost, p->stream));
            CK(cudaStreamSynchronize(p->stream));
        }
    }
    return 0;
}

int alloc_rej(clairplan_plan* p, uint32_t E) {
    bool ok = true;
    need<uint32_t>(p->rej_flag, E, ok);
    need<uint32_t>(p->rej_step, (uint64_t)E * kRejCap, ok);
    need<uint32_t>(p->rej_cum, (uint64_t)E * kRejCap, ok);
    need<uint32_t>(p->rej_count, E, ok);
    if (!ok) return fail(CLAIRPLAN_ENOMEM, "device allocation failed (rejection tables)");
    if (p->rej_count_h.size() != E) {
        p->rej_step_h.assign((size_t)E * kRejCap, 0);
        p->rej_cum_h.assign((size_t)E * kRejCap, 0);
        p->rej_count_h.assign(E, 0);
        CK(cudaMemsetAsync(p->rej_count.get<uint32_t>(), 0, E * sizeof(uint32_t), p->stream));
    }
    CK(cudaMemsetAsync(p->rej_flag.get<uint32_t>(), 0, E * sizeof(uint32_t), p->stream));
    return 0;
}

int ensure_ws(clairplan_plan* p, uint64_t n_elems, uint32_t nseg) {
    // radix tables: 256 x (n/2048 + nseg + 1) x (4 + 8) B, first-fit chunk arrays, scans
    const uint64_t tiles = n_elems / kRadixTile + nseg + 2;
    const uint64_t bytes = 256ull * tiles * 12 * 2 + (n_elems / 1024 + nseg + 2) * 96 +
                           (uint64_t)nseg * 64 + (64ull << 20);
    if (!p->wsbuf.ensure(bytes)) return fail(CLAIRPLAN_ENOMEM, "device allocation failed (workspace)");
    p->ws.base = p->wsbuf.get<char>();
    p->ws.cap = p->wsbuf.bytes;
    p->ws.used = 0;
    p->ws.overflow = false;
    return 0;
}

// K5-K8 on candidates (cand_k, cand_info: count<<16|rank) grouped per worker (wbeg/wlen).
int assign_tiers(clairplan_plan* p) {
    const uint32_t J = p->cfg.num_classes, nloc = p->nloc, F = p->part.F;
    const uint64_t D = p->D;
    cudaStream_t s = p->stream;
    bool ok = true;
    uint8_t* cand_cls = need<uint8_t>(p->cand_cls, D, ok);
    uint32_t* order = need<uint32_t>(p->order, D, ok);
    double* ssize = need<double>(p->sorted_size, D, ok);
    uint32_t* keys = need<uint32_t>(p->keys, D, ok);
    uint32_t* vals = need<uint32_t>(p->vals, D, ok);
    uint32_t* okeys = need<uint32_t>(p->okeys, D, ok);
    uint32_t* ovals = need<uint32_t>(p->ovals, D, ok);
    uint8_t* taken = need<uint8_t>(p->taken, D, ok);
    double* seqsz = need<double>(p->seqsz, D, ok);
    uint32_t* dest = need<uint32_t>(p->dest, D, ok);
    uint32_t* centries = need<uint32_t>(p->class_entries, D, ok);
    uint64_t* cstart = need<uint64_t>(p->class_start, (uint64_t)nloc * (J + 1), ok);
    uint64_t* clen = need<uint64_t>(p->class_len, (uint64_t)nloc * (J + 1), ok);
    uint32_t* htmp = need<uint32_t>(p->holders_tmp, 3 * D, ok);
    if (!ok) return fail(CLAIRPLAN_ENOMEM, "device allocation failed (tier assignment)");
    if (int rc = ensure_ws(p, D, nloc)) return rc;
    Workspace& ws = p->ws;
    const uint64_t* wbeg = p->wbeg.get<uint64_t>();
    const uint64_t* wlen = p->wlen.get<uint64_t>();
    const uint32_t* cand_k = p->cand_k.get<uint32_t>();
    const uint32_t* cand_info = p->cand_info.get<uint32_t>();

    TileMap tm;
    build_tilemap(s, wlen, nloc, D, kRadixTile, tm, ws);
    // K5: tier order
    const uint32_t maxc = p->generic ? p->maxcount : p->part.E;
    if (p->generic) launch_generic_count_keys(s, cand_info, D, maxc, keys);
    else launch_count_keys(s, cand_info, D, maxc, keys);
    {
        const uint32_t* kin = keys;
        const uint32_t* vin = nullptr;
        uint32_t passes = 0;
        for (uint32_t shift = 0; shift == 0 || ((uint64_t)maxc >> shift) != 0; shift += 8) {
            uint32_t* ko = (passes & 1) ? keys : okeys;
            uint32_t* vo = (passes & 1) ? vals : ovals;
            const size_t m = ws.mark();
            radix_pass(s, tm, wbeg, wlen, kin, vin, shift, ko, vo, nullptr, nullptr, ws);
            ws.release(m);
            kin = ko;
            vin = vo;
            ++passes;
            p->launches += 5;
        }
        CK(cudaMemcpyAsync(order, vin, D * sizeof(uint32_t), cudaMemcpyDeviceToDevice, s));
    }
    launch_gather_sizes(s, order, cand_k, p->sizes.get<double>(), D, ssize);
    CK(cudaMemsetAsync(cand_cls, 0, D, s));
    p->launches += 2;
    p->mark(5);

    // K6: first fit, class by class
    uint64_t* sb = ws.scratch<uint64_t>(nloc);
    uint64_t* sl = ws.scratch<uint64_t>(nloc);
    CK(cudaMemcpyAsync(sb, wbeg, nloc * sizeof(uint64_t), cudaMemcpyDeviceToDevice, s));
    CK(cudaMemcpyAsync(sl, wlen, nloc * sizeof(uint64_t), cudaMemcpyDeviceToDevice, s));
    const uint32_t* seq_idx = nullptr;  // pass 1: identity over the tier order
    const double* seq_sz = ssize;
    uint32_t* idx_buf[2] = {vals, ovals};
    for (uint32_t j = 1; j <= J; ++j) {
        if (j > 1) {
            // rejects of the previous pass, still in tier order
            launch_reject_keys(s, taken, D, seq_idx, keys, j % 2 ? idx_buf[0] : idx_buf[1]);
            const size_t m = ws.mark();
            TileMap tj;
            build_tilemap(s, sl, nloc, D, kRadixTile, tj, ws);
            uint64_t* sc = nullptr;
            uint32_t* nidx = j % 2 ? idx_buf[1] : idx_buf[0];
            radix_pass(s, tj, sb, sl, keys, j % 2 ? idx_buf[0] : idx_buf[1], 0, okeys, nidx,
                       nullptr, &sc, ws);
            uint64_t* nb = ws.scratch<uint64_t>(2 * (uint64_t)nloc);
            radix_regions(s, tj, sb, sl, sc, 1, nb, nb + nloc);
            CK(cudaMemcpyAsync(sb, nb, nloc * sizeof(uint64_t), cudaMemcpyDeviceToDevice, s));
            CK(cudaMemcpyAsync(sl, nb + nloc, nloc * sizeof(uint64_t), cudaMemcpyDeviceToDevice, s));
            ws.release(m);
            launch_gather_seq_sizes(s, nidx, ssize, sb, sl, nloc, seqsz);
            seq_idx = nidx;
            seq_sz = seqsz;
            p->launches += 10;
        }
        CK(cudaMemsetAsync(taken, 0, D, s));
        const size_t m = ws.mark();
        first_fit_pass(s, sb, sl, nloc, D, seq_sz, p->caps[j - 1], taken, ws);
        ws.release(m);
        launch_apply_pass(s, taken, D, seq_idx, order, (uint8_t)j, cand_cls);
        p->launches += 10;
    }

    p->mark(6);
    // K7: class lists = stable partition of first-access order by class
    launch_class_keys(s, cand_cls, D, J, keys);
    uint64_t* sc = nullptr;
    radix_pass(s, tm, wbeg, wlen, keys, cand_k, 0, okeys, centries, dest, &sc, ws);
    radix_regions(s, tm, wbeg, wlen, sc, J + 1, cstart, clen);
    p->launches += 7;
    p->mark(7);
    p->class_start_h.resize((size_t)nloc * (J + 1));
    p->class_len_h.resize((size_t)nloc * (J + 1));
    CK(cudaMemcpyAsync(p->class_start_h.data(), cstart, p->class_start_h.size() * 8,
                       cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(p->class_len_h.data(), clen, p->class_len_h.size() * 8,
                       cudaMemcpyDeviceToHost, s));

    if (p->generic) return generic_holders(p);
    // K8: holders at their pair slots
    launch_holder_scatter(s, cand_k, cand_info, cand_cls, dest, wbeg, wlen, cstart, J, nloc,
                          p->part.wbegin, p->pair_off.get<uint64_t>(), htmp);
    ++p->launches;
    CK(cudaStreamSynchronize(s));
    if (ws.overflow) return fail(CLAIRPLAN_ENOMEM, "internal workspace overflow");
    uint64_t H = 0;
    for (uint32_t w = 0; w < nloc; ++w)
        for (uint32_t d = 0; d < J; ++d) H += p->class_len_h[(size_t)w * (J + 1) + d];
    p->H = H;
    if (H == D) {
        p->holder_off_dev = p->pair_off.get<uint64_t>();
        p->holders_dev = htmp;
    } else {
        uint32_t* hc = need<uint32_t>(p->hcount, F, ok);
        uint64_t* ho = need<uint64_t>(p->hoff, (uint64_t)F + 1, ok);
        uint32_t* hl = need<uint32_t>(p->holders, 3 * std::max<uint64_t>(H, 1), ok);
        if (!ok) return fail(CLAIRPLAN_ENOMEM, "device allocation failed (holders)");
        launch_holder_count(s, p->pair_off.get<uint64_t>(), F, htmp, hc);
        exclusive_scan(s, hc, F, ho, ws);
        launch_holder_compact(s, p->pair_off.get<uint64_t>(), F, htmp, ho, hl);
        p->launches += 5;
        p->holder_off_dev = ho;
        p->holders_dev = hl;
    }
    return 0;
}

int build_seed_path(clairplan_plan* p) {
    cudaStream_t s = p->stream;
    const Part& part = p->part;
    const uint32_t F = part.F, E = part.E, nloc = p->nloc;
    bool ok = true;
    uint32_t* stream_buf = need<uint32_t>(p->stream_buf, p->A, ok);
    uint32_t* info = need<uint32_t>(p->info, (uint64_t)E * part.Fp, ok);  // pitched rows
    uint32_t* pcount = need<uint32_t>(p->pair_count, F, ok);
    uint64_t* poff = need<uint64_t>(p->pair_off, (uint64_t)F + 1, ok);
    uint32_t* segcnt = need<uint32_t>(p->segcnt, (uint64_t)nloc * E, ok);
    uint64_t* segoff = need<uint64_t>(p->seg_off, (uint64_t)nloc * E + 1, ok);
    uint64_t* wbeg = need<uint64_t>(p->wbeg, nloc, ok);
    uint64_t* wlen = need<uint64_t>(p->wlen, nloc, ok);
    if (!ok) return fail(CLAIRPLAN_ENOMEM, "device allocation failed (streams / histograms)");
    if (int rc = ensure_ws(p, std::max<uint64_t>((uint64_t)nloc * E, F), nloc)) return rc;
    if (int rc = alloc_rej(p, E)) return rc;
    uint32_t hs, nw, warps;
    size_t smem;
    if (sample_pass_config(part, &hs, &nw, &warps, &smem))
        return fail(CLAIRPLAN_EINVAL, "epochs/workers too large for the device histogram");

    for (int attempt = 0; attempt < 3; ++attempt) {
        p->launches = 0;
        CK(cudaEventRecord(p->ev0, s));
        p->mark(0);
        // K1-K3
        if (int rc = enqueue_perms(p, stream_buf, info, nullptr, 0, E)) return rc;
        p->mark(1);
        // K4a
        launch_sample_pass(s, part, info, pcount, hs, nw, warps, smem);
        exclusive_scan(s, pcount, F, poff, p->ws);
        p->mark(2);
        // K4b
        launch_seg_count(s, part, stream_buf, info, segcnt);
        exclusive_scan(s, segcnt, (uint64_t)nloc * E, segoff, p->ws);
        p->mark(3);
        p->launches += 8;
        std::vector<uint32_t> flags(E);
        uint64_t D = 0;
        CK(cudaMemcpyAsync(&D, segoff + (uint64_t)nloc * E, sizeof(uint64_t),
                           cudaMemcpyDeviceToHost, s));
        CK(cudaMemcpyAsync(flags.data(), p->rej_flag.get<uint32_t>(), E * sizeof(uint32_t),
                           cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        bool any = false;
        if (int rc = resolve_rejections(p, flags, &any)) return rc;
        if (any) continue;  // rebuild with the completed rejection tables
        p->D = D;
        if (D >= 0xFFFFFFFFull)
            return fail(CLAIRPLAN_EOVERFLOW, "more than 2^32-1 (worker, sample) pairs in one handle; "
                                             "shard the workers over several handles");
        uint32_t* ck = need<uint32_t>(p->cand_k, D, ok);
        uint32_t* ci = need<uint32_t>(p->cand_info, D, ok);
        if (!ok) return fail(CLAIRPLAN_ENOMEM, "device allocation failed (candidates)");
        launch_seg_write(s, part, stream_buf, info, segoff, ck, ci);
        launch_worker_segments(s, segoff, nloc, E, wbeg, wlen);
        p->launches += 2;
        p->mark(4);
        if (p->cfg.num_classes > 0) {
            if (int rc = assign_tiers(p)) return rc;
        } else {
            p->H = 0;
            uint64_t* ho = need<uint64_t>(p->hoff, (uint64_t)F + 1, ok);
            if (!ok) return fail(CLAIRPLAN_ENOMEM, "device allocation failed");
            CK(cudaMemsetAsync(ho, 0, ((uint64_t)F + 1) * 8, s));
            p->holder_off_dev = ho;
            p->holders_dev = nullptr;
            p->class_start_h.assign(nloc, 0);
            p->class_len_h.assign(nloc, 0);
        }
        if (p->cfg.num_classes == 0)
            for (int i = 5; i < clairplan_plan::kStages; ++i) p->mark(i);
        p->mark(clairplan_plan::kStages);
        CK(cudaEventRecord(p->ev1, s));
        CK(cudaEventSynchronize(p->ev1));
        CK(cudaGetLastError());
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, p->ev0, p->ev1));
        p->device_ms = ms;
        for (int i = 0; i < clairplan_plan::kStages; ++i) {
            float t = 0;
            if (p->sev[i] && p->sev[i + 1]) cudaEventElapsedTime(&t, p->sev[i], p->sev[i + 1]);
            p->stage_ms[i] = t;
        }
        p->built = true;
        return 0;
    }
    return fail(CLAIRPLAN_ECUDA, "rejection tables did not converge");
}

}  // namespace clairplan

// ---------------------------------------------------------------------------------------
namespace clairplan {

// ---- v2 seed path --------------------------------------------------------------------
bool v2_ok(const clairplan_plan* p) {
    const Part& part = p->part;
    return (p->nloc <= 65535) && part.E <= 1024 && p->cfg.num_classes <= 12 &&
           (uint64_t)p->nloc * part.E * part.E <= (1ull << 28);
}

// The whole-worker fit test of the all-fit path (allfit_decide_kernel) against capacity C,
// on the per-worker sums of the last seed build: sizes non-negative and every worker's total
// below C by more than any summation / chain rounding.  Then `s <= remaining` holds at every
// step of the chain of any subset of a worker's candidates in any order.
bool class_takes_all(const clairplan_plan* p, double C) {
    if (!p->sums_ok || p->wcnt_h.size() != (size_t)p->nloc + 1 || p->wcnt_h[p->nloc]) return false;
    for (uint32_t w = 0; w < p->nloc; ++w) {
        if (p->wcnt_h[w] == 0) continue;
        const double sw = (double)p->wsum_h[w] * 0x1.0p-20;
        const double tol = ((double)p->wcnt_h[w] + 1024.0) * std::max(C, sw) * 0x1.0p-48;
        if (!(C - sw > tol)) return false;
    }
    return true;
}

// First fit of the tier-ordered sizes, class by class (pack_first_fit, policies.cpp:40-55);
// cls[s] = class of tier-ordered element s (0 = not cached).
int first_fit_classes(clairplan_plan* p, const double* ssize, uint8_t* cls) {
    const uint32_t J = p->cfg.num_classes, nloc = p->nloc;
    const uint64_t D = p->D;
    cudaStream_t s = p->stream;
    Workspace& ws = p->ws;
    bool ok = true;
    unsigned long long* cnt = need<unsigned long long>(p->counters, 4, ok);
    if (!ok) return fail(CLAIRPLAN_ENOMEM, "device allocation failed (first fit)");
    CK(cudaMemsetAsync(cls, 0, D, s));
    uint64_t* sb = ws.scratch<uint64_t>(nloc);
    uint64_t* sl = ws.scratch<uint64_t>(nloc);
    CK(cudaMemcpyAsync(sb, p->wbeg.get<uint64_t>(), nloc * 8, cudaMemcpyDeviceToDevice, s));
    CK(cudaMemcpyAsync(sl, p->wlen.get<uint64_t>(), nloc * 8, cudaMemcpyDeviceToDevice, s));
    const uint32_t* seq_idx = nullptr;
    const double* seq_sz = ssize;
    const uint8_t* prev_taken = cls;  // class 1 writes its flags straight into cls (0/1)
    uint64_t remaining = D, prev_total = D;
    p->h_known = false;
    for (uint32_t j = 1; j <= J; ++j) {
        if (remaining == 0) {
            p->h_known = true;  // classes < j took every candidate
            break;
        }
        if (j > 1 && class_takes_all(p, p->caps[j - 1])) {
            // every worker's whole candidate set fits class j: its first-fit chain over the
            // rejects of classes < j takes all of them (policies.cpp:40-55, any order)
            launch_fill_class(s, cls, D, (uint8_t)j);
            ++p->launches;
            p->h_known = true;
            break;
        }
        uint8_t* taken = cls;
        if (j > 1) {
            // rejects of the previous class, still in tier order, packed for this class
            taken = need<uint8_t>(p->taken, D, ok);
            uint32_t* ib0 = need<uint32_t>(p->vals, remaining, ok);
            uint32_t* ib1 = need<uint32_t>(p->ovals, remaining, ok);
            double* seqsz = need<double>(p->seqsz, remaining, ok);
            if (!ok) return fail(CLAIRPLAN_ENOMEM, "device allocation failed (first fit)");
            uint32_t* out_idx = (j % 2) ? ib1 : ib0;
            const size_t m = ws.mark();
            uint64_t* nb = ws.scratch<uint64_t>(2 * (uint64_t)nloc);
            compact_rejects(s, sb, sl, nloc, prev_total, prev_taken, seq_idx, ssize, 0, out_idx,
                            seqsz, nb, nb + nloc, ws);
            CK(cudaMemcpyAsync(sb, nb, nloc * 8, cudaMemcpyDeviceToDevice, s));
            CK(cudaMemcpyAsync(sl, nb + nloc, nloc * 8, cudaMemcpyDeviceToDevice, s));
            ws.release(m);
            seq_idx = out_idx;
            seq_sz = seqsz;
            CK(cudaMemsetAsync(taken, 0, remaining, s));
            p->launches += 7;
        }
        CK(cudaMemsetAsync(cnt, 0, 8, s));
        const size_t m = ws.mark();
        const uint64_t total = (j == 1) ? D : remaining;
        const bool gather = j == 1 && p->ssize_pending;  // tier-order sizes not written yet
        first_fit_pass(s, sb, sl, nloc, total, seq_sz, p->caps[j - 1], taken, ws, cnt,
                       gather ? p->sorted_k.get<uint32_t>() : nullptr,
                       gather ? p->sizes.get<double>() : nullptr);
        if (gather) p->ssize_pending = false;
        ws.release(m);
        p->launches += 6;
        if (j > 1) {
            launch_apply_pass(s, taken, remaining, seq_idx, nullptr, (uint8_t)j, cls);
            ++p->launches;
        }
        prev_taken = taken;
        prev_total = total;
        if (j < J) {
            unsigned long long t = 0;
            CK(cudaMemcpyAsync(&t, cnt, 8, cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
            remaining -= t;
        }
    }
    return 0;
}


// (count at first access) source of the segment passes: info[e][k] (dense sample pass) or
// einfo[csr slot] with cpos[stream index] = csr slot (sparse sample pass of a sharded handle)
inline const void* info_src(clairplan_plan* p) {
    return p->sparse ? p->einfo.get<uint16_t>() : p->info16.get<void>();
}

int holders_v2(clairplan_plan* p);
int no_classes_v2(clairplan_plan* p);

// holder records from the [E][F] class/position rows (tier.cu): dense sample-major arrays,
// classes and list positions fit 4 + 28 bits
bool hp_path_ok(const clairplan_plan* p) {
    const Part& part = p->part;
    uint64_t lmax = 0;
    for (uint32_t w : {part.wbegin, part.wend - 1}) lmax = std::max<uint64_t>(lmax, part.E * part.epoch_len(w));
    // (hp_fill + holder_hp: 12.5 + 8.3 ms against holder_tile's 30 ms at the ImageNet-22k
    // shape, round-2 launch lists; CLAIRPLAN_NO_HP_PATH=1: A/B)
    static const bool on = !ab_flag("CLAIRPLAN_NO_HP_PATH");
    return on && !p->sparse && !p->allfit && p->cfg.num_classes <= 15 && lmax < (1ull << 28) &&
           holder_hp_ok(part);
}

// K6-K8 of the v2 path on the cached tier-ordered sizes / block masks: first fit, block class
// records, class lists, holder CSR.  Also the whole of clairplan_reassign.
int assign_v2(clairplan_plan* p) {
    cudaStream_t s = p->stream;
    const Part& part = p->part;
    const uint32_t E = part.E, nloc = p->nloc, J = p->cfg.num_classes;
    const uint32_t MB = p->v2_mb;
    const uint64_t nblk = p->v2_nblk;
    const uint64_t D = p->D;
    uint32_t np = 0;
    while ((1u << np) <= J) ++np;
    bool ok = true;
    uint32_t* stream_buf = p->stream_buf.get<uint32_t>();
    uint32_t* bmask = p->blkmask.get<uint32_t>();
    uint32_t* bbase = p->blkbase.get<uint32_t>();
    uint32_t* dest = p->dest.get<uint32_t>();
    double* ssize = p->sorted_size.get<double>();
    uint8_t* cls = need<uint8_t>(p->cand_cls, D, ok);
    uint32_t* centries = need<uint32_t>(p->class_entries, D, ok);
    const uint32_t Rp = ((np + J) + 3) & ~3u;
    uint32_t* rec = need<uint32_t>(p->planes, (uint64_t)std::max<uint32_t>(Rp, 4) * nblk, ok);
    uint32_t* cbase = need<uint32_t>(p->cbase, (uint64_t)nloc * std::max<uint32_t>(J, 1), ok);
    uint32_t* ccount = need<uint32_t>(p->ccount, std::max<uint32_t>(J, 1) * nblk, ok);
    uint64_t* cpre = need<uint64_t>(p->cpre, std::max<uint32_t>(J, 1) * (nblk + 1), ok);
    uint64_t* clen = need<uint64_t>(p->class_len, (uint64_t)nloc * std::max<uint32_t>(J, 1), ok);
    uint64_t* cstart = need<uint64_t>(p->class_start, (uint64_t)nloc * std::max<uint32_t>(J, 1) + 1, ok);
    if (!ok) return fail(CLAIRPLAN_ENOMEM, "device allocation failed (tier assignment)");
    if (J > 0) {
        // K6: first fit class by class
        if (int rc = first_fit_classes(p, ssize, cls)) return rc;
        p->mark(6);
        // K7: block class records, class lists
        launch_blk_codes(s, part, MB, bmask, bbase, dest, cls, np, J, Rp, rec, ccount, nblk);
        for (uint32_t j = 0; j < J; ++j)
            exclusive_scan(s, ccount + (uint64_t)j * nblk, nblk, cpre + (uint64_t)j * (nblk + 1), p->ws);
        launch_rec_fill(s, cpre, nblk, np, J, Rp, rec, nloc, E, MB, cbase);
        launch_class_lens(s, nloc, E, MB, J, cpre, nblk, clen);
        exclusive_scan(s, clen, (uint64_t)nloc * J, cstart, p->ws);
        launch_class_write(s, part, MB, stream_buf, rec, np, J, Rp, cbase, cstart, centries, nblk);
        // build_export: when every candidate is cached (H = D, known here) the class lists are
        // final and contiguous: copy them out behind the stream copy while the holders build
        static const bool early_cl = ab_knob("CLAIRPLAN_EARLY_CL", 1) != 0;  // A/B
        if (early_cl && p->x_class && p->h_known && D <= p->x_class_cap && p->xstream) {
            CK(cudaEventRecord(p->xev, s));
            CK(cudaStreamWaitEvent(p->xstream, p->xev, 0));
            CK(cudaMemcpyAsync(p->x_class, centries, D * 4, cudaMemcpyDeviceToHost, p->xstream));
            p->x_class_done = true;
        }
        p->hp_path = hp_path_ok(p);
        if (p->hp_path) {
            uint32_t* hp = need<uint32_t>(p->hpos, (uint64_t)E * part.Fp, ok);
            if (!ok) return fail(CLAIRPLAN_ENOMEM, "device allocation failed (holder positions)");
            uint32_t* claim = need<uint32_t>(p->sched, 8, ok);
            if (!ok) return fail(CLAIRPLAN_ENOMEM, "device allocation failed (holder positions)");
            launch_hp_fill(s, part, p->inv.get<uint32_t>(), p->rank16.get<uint16_t>(), MB, rec, np, J, Rp,
                           cbase, hp, claim + 1);
            ++p->launches;
        }
        p->launches += 4 + 3 * J + 3;
        p->cl_contig = true;
        return holders_v2(p);
    }
    return no_classes_v2(p);
}

// K8 and the host-side class-list geometry, after the block records, class bases and class
// lists exist (general path or all-fit path).
int holders_v2(clairplan_plan* p) {
    cudaStream_t s = p->stream;
    const Part& part = p->part;
    const uint32_t F = part.F, nloc = p->nloc, J = p->cfg.num_classes;
    const uint64_t D = p->D;
    uint32_t np = 0;
    while ((1u << np) <= J) ++np;
    const uint32_t Rp = ((np + J) + 3) & ~3u;
    bool ok = true;
    uint32_t* inv = p->inv.get<uint32_t>();
    uint16_t* rank16 = p->rank16.get<uint16_t>();
    uint64_t* poff = p->pair_off.get<uint64_t>();
    uint32_t* htmp = need<uint32_t>(p->holders_tmp, 3 * D, ok);
    uint32_t* rec = p->planes.get<uint32_t>();
    uint32_t* cbase = p->cbase.get<uint32_t>();
    uint64_t* clen = p->class_len.get<uint64_t>();
    uint64_t* cstart = p->class_start.get<uint64_t>();
    const uint32_t MB = p->v2_mb;
    if (!ok) return fail(CLAIRPLAN_ENOMEM, "device allocation failed (holders)");
    {
        std::vector<uint64_t> hlen((size_t)nloc * J), hst((size_t)nloc * J);
        CK(cudaMemcpyAsync(hlen.data(), clen, hlen.size() * 8, cudaMemcpyDeviceToHost, s));
        CK(cudaMemcpyAsync(hst.data(), cstart, hst.size() * 8, cudaMemcpyDeviceToHost, s));
        p->mark(7);
        // K8: holder CSR, sample-major
        if (p->sparse)
            launch_holder_sparse(s, part, p->A, p->soff.get<uint64_t>(), p->stream_buf.get<uint32_t>(),
                                 p->csr.get<uint32_t>(), p->erank.get<uint16_t>(), MB, rec, np, J, Rp,
                                 cbase, poff, htmp, p->allfit);
        else if (p->hp_path && !p->allfit)
            launch_holder_hp(s, part, inv, rank16, p->hpos.get<uint32_t>(), poff, htmp);
        else
            launch_holder_tile(s, part, inv, rank16, MB, rec, np, J, Rp, cbase, poff, htmp, p->allfit);
        ++p->launches;
        CK(cudaStreamSynchronize(s));
        p->class_start_h.assign((size_t)nloc * (J + 1), 0);
        p->class_len_h.assign((size_t)nloc * (J + 1), 0);
        uint64_t H = 0;
        for (uint32_t w = 0; w < nloc; ++w)
            for (uint32_t j = 0; j < J; ++j) {
                p->class_start_h[(size_t)w * (J + 1) + j] = hst[(size_t)w * J + j];
                p->class_len_h[(size_t)w * (J + 1) + j] = hlen[(size_t)w * J + j];
                H += hlen[(size_t)w * J + j];
            }
        p->H = H;
        if (H == D) {
            p->holder_off_dev = poff;
            p->holders_dev = htmp;
        } else {
            uint32_t* hc = need<uint32_t>(p->hcount, F, ok);
            uint64_t* ho = need<uint64_t>(p->hoff, (uint64_t)F + 1, ok);
            uint32_t* hl = need<uint32_t>(p->holders, 3 * std::max<uint64_t>(H, 1), ok);
            if (!ok) return fail(CLAIRPLAN_ENOMEM, "device allocation failed (holders)");
            launch_holder_count(s, poff, F, htmp, hc);
            exclusive_scan(s, hc, F, ho, p->ws);
            launch_holder_compact(s, poff, F, htmp, ho, hl);
            p->launches += 5;
            p->holder_off_dev = ho;
            p->holders_dev = hl;
        }
    }
    return 0;
}

int no_classes_v2(clairplan_plan* p) {
    cudaStream_t s = p->stream;
    const uint32_t F = p->part.F, nloc = p->nloc;
    bool ok = true;
    {
        p->H = 0;
        uint64_t* ho = need<uint64_t>(p->hoff, (uint64_t)F + 1, ok);
        if (!ok) return fail(CLAIRPLAN_ENOMEM, "device allocation failed");
        CK(cudaMemsetAsync(ho, 0, ((uint64_t)F + 1) * 8, s));
        p->holder_off_dev = ho;
        p->holders_dev = nullptr;
        p->class_start_h.assign(nloc, 0);
        p->class_len_h.assign(nloc, 0);
        p->mark(6);
        p->mark(7);
    }
    return 0;
}


// K4c: every candidate's first-order index -> tier position (dest), the sizes in tier order,
// the block first-masks; per-worker candidate ranges (wbeg / wlen).
int tier_order_v2(clairplan_plan* p) {
    cudaStream_t s = p->stream;
    const Part& part = p->part;
    const uint32_t E = part.E, nloc = p->nloc;
    const uint64_t D = p->D;
    bool ok = true;
    uint32_t* dest = need<uint32_t>(p->dest, D, ok);
    double* ssize = need<double>(p->sorted_size, D, ok);
    if (!ok) return fail(CLAIRPLAN_ENOMEM, "device allocation failed (candidates)");
    const uint64_t* segoff = p->seg_off.get<uint64_t>();
    if (!p->hist_ready) {  // all-fit build: the count histograms were not needed then
        const uint64_t NEE = (uint64_t)nloc * E * E;
        launch_seg_hist(s, part, p->stream_buf.get<uint32_t>(), info_src(p), p->info8, p->sparse ? p->cpos.get<uint32_t>() : nullptr,
                        p->seghist.get<uint32_t>(), p->segcnt.get<uint32_t>());
        exclusive_scan(s, p->seghist.get<uint32_t>(), NEE, p->sorted_base.get<uint64_t>(), p->ws);
        exclusive_scan(s, p->segcnt.get<uint32_t>(), (uint64_t)nloc * E, p->seg_off.get<uint64_t>(), p->ws);
        p->launches += 4;
        p->hist_ready = true;
    }
    if (p->sparse) {
        launch_seg_write2(s, part, p->stream_buf.get<uint32_t>(), p->einfo.get<uint16_t>(), p->cpos.get<uint32_t>(),
                          p->sizes.get<double>(), segoff, p->sorted_base.get<uint64_t>(), p->v2_mb, dest,
                          ssize, p->blkmask.get<uint32_t>(), p->blkbase.get<uint32_t>());
    } else {  // epoch-major segment CTAs, then the size gather on its own (tier.cu)
        uint32_t* sk = need<uint32_t>(p->sorted_k, D, ok);
        if (!ok) return fail(CLAIRPLAN_ENOMEM, "device allocation failed (tier order)");
        uint32_t* claim = need<uint32_t>(p->sched, 8, ok);
        if (!ok) return fail(CLAIRPLAN_ENOMEM, "device allocation failed (tier order)");
        launch_seg_write3(s, part, p->stream_buf.get<uint32_t>(), info_src(p), p->info8, segoff,
                          p->sorted_base.get<uint64_t>(), p->v2_mb, dest, sk,
                          p->blkmask.get<uint32_t>(), p->blkbase.get<uint32_t>(), claim);
        p->ssize_pending = true;  // gathered by class 1's first-fit statistics pass
    }
    launch_worker_segments(s, segoff, nloc, E, p->wbeg.get<uint64_t>(), p->wlen.get<uint64_t>());
    p->launches += 2;
    p->tier_ready = true;
    return 0;
}

// Speculative all-fit pipeline: launched before the host knows the fit test's outcome (it is
// computed on the device into *gate); every kernel exits at once when the test failed, and the
// host then runs the tier path.  Buffers are sized by A >= D (D is not known yet).
int spec_allfit_launch(clairplan_plan* p, const uint32_t* gate) {
    cudaStream_t s = p->stream;
    const Part& part = p->part;
    const uint32_t E = part.E, nloc = p->nloc, J = p->cfg.num_classes;
    uint32_t np = 0;
    while ((1u << np) <= J) ++np;
    const uint32_t Rp = ((np + J) + 3) & ~3u;
    const uint32_t C = (uint32_t)((part.epoch_len(part.wbegin) + kAllfitChunk - 1) / kAllfitChunk);
    bool ok = true;
    uint32_t* centries = need<uint32_t>(p->class_entries, p->A, ok);
    uint32_t* rec = need<uint32_t>(p->planes, (uint64_t)std::max<uint32_t>(Rp, 4) * p->v2_nblk, ok);
    uint32_t* cbase = need<uint32_t>(p->cbase, (uint64_t)nloc * J, ok);
    uint64_t* clen = need<uint64_t>(p->class_len, (uint64_t)nloc * J, ok);
    uint64_t* cstart = need<uint64_t>(p->class_start, (uint64_t)nloc * J + 1, ok);
    unsigned long long* status = need<unsigned long long>(p->chstatus, (uint64_t)nloc * E * C, ok);
    uint32_t* ticket = need<uint32_t>(p->counters, 4, ok);
    uint32_t* htmp = need<uint32_t>(p->holders_tmp, 3 * std::max<uint64_t>(p->A, 1), ok);
    if (!ok) return fail(CLAIRPLAN_ENOMEM, "device allocation failed (all-fit)");
    // stage labels: the one segment pass writes the class lists (stage 6), the first fit is
    // decided by the whole-worker test (no tier order, no first-fit chain)
    p->mark(3);
    p->mark(4);
    p->mark(5);
    p->mark(6);
    launch_seg_allfit(s, part, p->stream_buf.get<uint32_t>(), info_src(p), p->info8,
                      p->sparse ? p->cpos.get<uint32_t>() : nullptr, p->v2_mb, C, status, ticket,
                      rec, centries, gate);
    launch_allfit_meta(s, part, J, p->wcnt.get<uint32_t>(), clen, cstart, cbase, gate);
    p->mark(7);
    const uint64_t* poff = p->pair_off.get<uint64_t>();
    if (p->sparse)
        launch_holder_sparse(s, part, p->A, p->soff.get<uint64_t>(), p->stream_buf.get<uint32_t>(),
                             p->csr.get<uint32_t>(), p->erank.get<uint16_t>(), p->v2_mb, rec, np, J,
                             Rp, cbase, poff, htmp, true, gate);
    else
        launch_holder_tile(s, part, p->inv.get<uint32_t>(), p->rank16.get<uint16_t>(), p->v2_mb, rec,
                           np, J, Rp, cbase, poff, htmp, true, gate);
    p->launches += 6;
    return 0;
}

// host state of a finished all-fit build: class list (w, 1) at the worker's stream offset with
// its candidate count, (w, j > 1) empty; every pair is a holder record
void finish_allfit(clairplan_plan* p, const std::vector<uint32_t>& wcnt_h) {
    const uint32_t nloc = p->nloc, J = p->cfg.num_classes;
    p->class_start_h.assign((size_t)nloc * (J + 1), 0);
    p->class_len_h.assign((size_t)nloc * (J + 1), 0);
    for (uint32_t w = 0; w < nloc; ++w) {
        const uint64_t a = p->part.stream_offset(p->part.wbegin + w);
        for (uint32_t j = 0; j < J; ++j) {
            p->class_start_h[(size_t)w * (J + 1) + j] = j == 0 ? a : a + wcnt_h[w];
            p->class_len_h[(size_t)w * (J + 1) + j] = j == 0 ? wcnt_h[w] : 0;
        }
    }
    p->H = p->D;
    p->holder_off_dev = p->pair_off.get<uint64_t>();
    p->holders_dev = p->holders_tmp.get<uint32_t>();
    p->cl_contig = false;
    p->allfit = true;
}

// sharded build from received streams: sparse (CSR) or dense sample-major passes
static bool sharded_sparse(clairplan_plan* p) {
    const char* dense_env = path_switch("CLAIRPLAN_DENSE");  // "1": dense, "0": sparse, unset: cost model
    return dense_env ? dense_env[0] == '0' && sparse_path_fits(p->part) : sparse_path_ok(p->part, p->A);
}

int build_seed_path_v2(clairplan_plan* p, const uint32_t* ext_perms,
                       const uint32_t* ext_streams = nullptr, const EpochSplit* es = nullptr) {
    cudaStream_t s = p->stream;
    const Part& part = p->part;
    const uint32_t F = part.F, E = part.E, nloc = p->nloc, J = p->cfg.num_classes;
    const uint32_t MB = (uint32_t)((part.epoch_len(part.wbegin) + 31) / 32);
    const uint64_t nblk = (uint64_t)nloc * E * MB;
    uint32_t np = 0;
    while ((1u << np) <= J) ++np;  // bits to hold classes 0..J
    const uint64_t NEE = (uint64_t)nloc * E * E;
    bool ok = true;
    // sparse sample-major passes (sharded handle fed by the all-to-all; CLAIRPLAN_DENSE=1: A/B)
    const bool sparse = ext_streams && sharded_sparse(p);
    uint32_t* stream_buf = need<uint32_t>(p->stream_buf, p->A, ok);
    p->hook_fired = false;
    bool hook_called = false;  // at most once per build: every rank calls its collective once
    // the dense [E][F] sample-major arrays (not needed by the sparse passes)
    uint32_t* inv = sparse ? nullptr : need<uint32_t>(p->inv, (uint64_t)E * part.Fp, ok);
    const uint64_t EFp = (uint64_t)E * part.Fp;  // pitched u16 rows
    // info rows are u8 when every count fits (E <= 255) and the tile sample pass writes them:
    // half the L2 footprint of the gathers from the segment passes
    static const bool lanes_only = ab_flag("CLAIRPLAN_SAMPLE_LANES");  // A/B
    const bool tile_pass = !sparse && tile_path_ok(part) && !lanes_only;
    p->info8 = tile_pass && E <= 255;
    void* info = sparse ? nullptr : need<uint8_t>(p->info16, EFp * (p->info8 ? 1 : 2), ok);
    uint16_t* rank16 = sparse ? nullptr : need<uint16_t>(p->rank16, EFp, ok);
    uint32_t* pcount = need<uint32_t>(p->pair_count, F, ok);
    uint64_t* poff = need<uint64_t>(p->pair_off, (uint64_t)F + 1, ok);
    uint32_t* seghist = need<uint32_t>(p->seghist, NEE, ok);
    uint64_t* sbase = need<uint64_t>(p->sorted_base, NEE + 1, ok);
    uint32_t* segcnt = need<uint32_t>(p->segcnt, (uint64_t)nloc * E, ok);
    uint64_t* segoff = need<uint64_t>(p->seg_off, (uint64_t)nloc * E + 1, ok);
    uint64_t* wbeg = need<uint64_t>(p->wbeg, nloc, ok);
    uint64_t* wlen = need<uint64_t>(p->wlen, nloc, ok);
    uint32_t* bmask = need<uint32_t>(p->blkmask, nblk, ok);
    uint32_t* bbase = need<uint32_t>(p->blkbase, nblk, ok);
    unsigned long long* wsum = need<unsigned long long>(p->wsum, nloc, ok);
    uint32_t* wcnt = need<uint32_t>(p->wcnt, (uint64_t)nloc + 1, ok);  // + the negative-size flag
    uint32_t* wneg = wcnt + nloc;
    p->sparse = sparse;
    uint32_t *sp_cnt = nullptr, *sp_cur = nullptr, *sp_csr = nullptr;
    uint64_t *sp_koff = nullptr, *sp_soff = nullptr;
    uint16_t *sp_einfo = nullptr, *sp_erank = nullptr;
    if (sparse) {
        sp_cnt = need<uint32_t>(p->hcount, F, ok);
        sp_cur = need<uint32_t>(p->sp_cur, F, ok);
        sp_koff = need<uint64_t>(p->koff, (uint64_t)F + 1, ok);
        sp_csr = need<uint32_t>(p->csr, p->A, ok);
        sp_soff = need<uint64_t>(p->soff, (uint64_t)nloc + 1, ok);
        sp_einfo = need<uint16_t>(p->einfo, p->A, ok);
        sp_erank = need<uint16_t>(p->erank, p->A, ok);
        need<uint32_t>(p->cpos, p->A, ok);
    }
    if (!ok) return fail(CLAIRPLAN_ENOMEM, "device allocation failed (streams / histograms)");
    if (int rc = ensure_ws(p, std::max<uint64_t>(p->A, std::max<uint64_t>(NEE, F)), nloc)) return rc;
    if (int rc = alloc_rej(p, E)) return rc;
    const bool lanes = lane_path_ok(part);

    for (int attempt = 0; attempt < 3; ++attempt) {
        p->launches = 0;
        p->ws.used = 0;
        CK(cudaEventRecord(p->ev0, s));
        p->mark(0);
        // K1-K3: permutations -> streams + inverse permutations
        if (ext_streams) {  // multi-GPU: epoch-range streams from every rank (all-to-all)
            launch_stream_relayout(s, part, *es, ext_streams, stream_buf);
            ++p->launches;
            if (!sparse) {
                launch_stream_inv(s, part, stream_buf, inv, p->inv_own_lo, p->inv_own_hi);
                ++p->launches;
            }
        } else if (ext_perms) {
            launch_perm_scatter(s, part, ext_perms, inv, stream_buf);
            ++p->launches;
        } else if (int rc = enqueue_perms(p, stream_buf, inv, nullptr, 0, E)) {
            return rc;
        }
        p->mark(1);
        if (p->x_streams) {
            // build_export: the streams are final (unless a Lemire rejection turns up at the
            // check below; the retry then issues a second copy behind this one on the same
            // stream), so copy them out while the rest of the plan builds
            CK(cudaEventRecord(p->xev, s));
            CK(cudaStreamWaitEvent(p->xstream, p->xev, 0));
            CK(cudaMemcpyAsync(p->x_streams, stream_buf, p->A * 4, cudaMemcpyDeviceToHost, p->xstream));
        }
        // K4a: per-sample (worker, count, first epoch)
        // Large F: the segment histograms are accumulated by the sample pass itself (REDs
        // overlap its latency); small F: a separate warp-per-segment pass is cheaper.
        static const bool red_ok = ab_knob("CLAIRPLAN_RED_HIST", 1) != 0;  // A/B
        const bool red_hist = F >= (1u << 22) && !sparse && red_ok;
        uint32_t* hist_out = red_hist ? seghist : nullptr;
        if (red_hist) CK(cudaMemsetAsync(seghist, 0, NEE * 4, s));
        // per-worker candidate size sums for the whole-worker fit test (all-fit path)
        const bool no_allfit = path_switch("CLAIRPLAN_NO_ALLFIT") != nullptr;
        const bool sums = J > 0 && !no_allfit && (sparse || (tile_path_ok(part) && !lanes_only));
        WorkerSums wsm;
        if (sums) {
            wsm.sizes = p->sizes.get<double>();
            wsm.sum = wsum;
            wsm.cnt = wcnt;
            wsm.neg = wneg;
            CK(cudaMemsetAsync(wsum, 0, (size_t)nloc * 8, s));
            CK(cudaMemsetAsync(wcnt, 0, (size_t)nloc * 4 + 4, s));  // wcnt and wneg
        }
        if (sparse) {
            launch_sparse_csr(s, part, stream_buf, p->A, sp_cnt, sp_koff, sp_cur, sp_csr,
                              p->cpos.get<uint32_t>(), sp_soff, p->ws);
            launch_sparse_sample(s, part, sp_soff, sp_koff, sp_csr, pcount, sp_einfo, sp_erank, wsm);
            p->launches += 7;
        } else if (tile_path_ok(part) && !lanes_only) {
            launch_sample_tile(s, part, inv, info, p->info8, rank16, pcount, hist_out, wsm);
        } else if (lanes) {
            launch_sample_lanes(s, part, inv, static_cast<uint16_t*>(info), rank16, pcount, hist_out);
        } else {
            launch_sample_hash(s, part, inv, static_cast<uint16_t*>(info), rank16, pcount, nullptr, nullptr, F, hist_out);
        }
        exclusive_scan(s, pcount, F, poff, p->ws);
        p->mark(2);
        if (p->hook_fn && !hook_called) {
            CK(cudaMemcpyAsync(p->hook_counts, pcount, (size_t)F * 4, cudaMemcpyDeviceToDevice, s));
            if (!p->hook_ev) CK(cudaEventCreateWithFlags(&p->hook_ev, cudaEventDisableTiming));
            CK(cudaEventRecord(p->hook_ev, s));
            CK(cudaStreamWaitEvent(p->hook_stream, p->hook_ev, 0));
            p->hook_fn(p->hook_user);
            hook_called = true;
            p->hook_fired = true;
        } else {
            p->hook_fired = false;  // a rejection rerun: the hooked counts are stale
        }
        // speculative all-fit pipeline (decided on the device, checked at the one sync below)
        uint32_t* gate = nullptr;
        if (sums) {
            gate = need<uint32_t>(p->allfit_gate, 1, ok);
            if (!ok) return fail(CLAIRPLAN_ENOMEM, "device allocation failed");
            launch_allfit_decide(s, nloc, wsum, wcnt, p->caps[0], gate);
            p->v2_mb = MB;
            p->v2_nblk = nblk;
            if (int rc = spec_allfit_launch(p, gate)) return rc;
        }
        std::vector<uint32_t> flags(E);
        uint64_t D = 0;
        uint32_t gate_h = 0;
        std::vector<uint32_t> hcnt(sums ? nloc : 0);
        CK(cudaMemcpyAsync(&D, poff + F, 8, cudaMemcpyDeviceToHost, s));
        if (sums) {
            CK(cudaMemcpyAsync(hcnt.data(), wcnt, (size_t)nloc * 4, cudaMemcpyDeviceToHost, s));
            CK(cudaMemcpyAsync(&gate_h, gate, 4, cudaMemcpyDeviceToHost, s));
            p->wsum_h.resize(nloc);
            p->wcnt_h.resize((size_t)nloc + 1);
            CK(cudaMemcpyAsync(p->wsum_h.data(), wsum, (size_t)nloc * 8, cudaMemcpyDeviceToHost, s));
            CK(cudaMemcpyAsync(p->wcnt_h.data(), wcnt, ((size_t)nloc + 1) * 4, cudaMemcpyDeviceToHost, s));
        }
        p->sums_ok = sums;
        CK(cudaMemcpyAsync(flags.data(), p->rej_flag.get<uint32_t>(), E * 4, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        bool any = false;
        if (int rc = resolve_rejections(p, flags, &any)) return rc;
        if (any) continue;
        if (D >= 0xFFFFFFFFull)
            return fail(CLAIRPLAN_EOVERFLOW, "more than 2^32-1 (worker, sample) pairs in one handle (" +
                                                 std::to_string(D) + " of " + std::to_string(p->A) +
                                                 " entries); shard the workers over several handles");
        const bool allfit = sums && gate_h != 0;
        if (allfit) {  // the speculative pipeline produced the plan
            p->D = D;
            p->v2_mb = MB;
            p->v2_nblk = nblk;
            p->tier_ready = false;
            p->hist_ready = false;
            finish_allfit(p, hcnt);
            p->launches += 10;
            p->mark(clairplan_plan::kStages);
            CK(cudaEventRecord(p->ev1, s));
            CK(cudaEventSynchronize(p->ev1));
            CK(cudaGetLastError());
            if (p->ws.overflow) return fail(CLAIRPLAN_ENOMEM, "internal workspace overflow");
            float ms = 0;
            CK(cudaEventElapsedTime(&ms, p->ev0, p->ev1));
            p->device_ms = ms;
            for (int i = 0; i < clairplan_plan::kStages; ++i) {
                float t = 0;
                if (p->sev[i] && p->sev[i + 1]) cudaEventElapsedTime(&t, p->sev[i], p->sev[i + 1]);
                p->stage_ms[i] = t;
            }
            p->v2 = true;
            p->built = true;
            return 0;
        }
        // tier path. K4b: per-segment count histograms -> first-order and tier-order bases
        if (red_hist) launch_segcnt(s, nloc, E, seghist, segcnt);
        else launch_seg_hist(s, part, stream_buf, info_src(p), p->info8, p->sparse ? p->cpos.get<uint32_t>() : nullptr, seghist, segcnt);
        exclusive_scan(s, seghist, NEE, sbase, p->ws);
        exclusive_scan(s, segcnt, (uint64_t)nloc * E, segoff, p->ws);
        p->hist_ready = true;
        p->mark(3);
        p->launches += 10;
        p->D = D;
        if (D >= 0xFFFFFFFFull)
            return fail(CLAIRPLAN_EOVERFLOW, "more than 2^32-1 (worker, sample) pairs in one handle; "
                                             "shard the workers over several handles");
        p->v2_mb = MB;
        p->v2_nblk = nblk;
        p->tier_ready = false;
        p->allfit = false;
        if (int rc = tier_order_v2(p)) return rc;
        p->mark(4);
        p->mark(5);
        if (int rc = assign_v2(p)) return rc;
        p->mark(clairplan_plan::kStages);
        CK(cudaEventRecord(p->ev1, s));
        CK(cudaEventSynchronize(p->ev1));
        CK(cudaGetLastError());
        if (p->ws.overflow) return fail(CLAIRPLAN_ENOMEM, "internal workspace overflow");
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, p->ev0, p->ev1));
        p->device_ms = ms;
        for (int i = 0; i < clairplan_plan::kStages; ++i) {
            float t = 0;
            if (p->sev[i] && p->sev[i + 1]) cudaEventElapsedTime(&t, p->sev[i], p->sev[i + 1]);
            p->stage_ms[i] = t;
        }
        p->v2 = true;
        p->built = true;
        return 0;
    }
    return fail(CLAIRPLAN_ECUDA, "rejection tables did not converge");
}

}  // namespace clairplan

extern "C" {

int clairplan_version(void) { return 1; }

const char* clairplan_last_error(void) { return g_err.c_str(); }

int clairplan_validate(const clairplan_config* c) {
    if (!c) return fail(CLAIRPLAN_EINVAL, "null config");
    return validate_partition(c->samples, c->num_workers, c->global_batch, c->epochs);
}

int clairplan_create(const clairplan_config* c, clairplan_t* out) {
    if (!c || !out) return fail(CLAIRPLAN_EINVAL, "null argument");
    *out = nullptr;
    if (int rc = validate_partition(c->samples, c->num_workers, c->global_batch, c->epochs))
        return rc;
    if (c->epochs > 65535) return fail(CLAIRPLAN_EINVAL, "device plan supports at most 65535 epochs");
    if (c->num_classes > 254) return fail(CLAIRPLAN_EINVAL, "device plan supports at most 254 cache classes");
    if (c->num_classes && !c->capacities_mb) return fail(CLAIRPLAN_EINVAL, "capacities_mb is null");
    if (!c->sizes_mb && c->num_classes) return fail(CLAIRPLAN_EINVAL, "sizes_mb is null");
    uint32_t wb = c->worker_begin, we = c->worker_end;
    if (wb == 0 && we == 0) we = c->num_workers;
    if (wb >= we || we > c->num_workers) return fail(CLAIRPLAN_EINVAL, "invalid worker range");
    if (int rc = check_device(c->device)) return rc;
    auto* p = new clairplan_plan();
    p->device = c->device;
    p->cfg = *c;
    p->cfg.worker_begin = wb;
    p->cfg.worker_end = we;
    p->caps.assign(c->capacities_mb, c->capacities_mb + c->num_classes);
    p->cfg.capacities_mb = nullptr;
    p->cfg.sizes_mb = nullptr;
    p->part = make_part(c->samples, c->num_workers, c->global_batch, c->epochs, c->drop_last != 0,
                        wb, we);
    p->nloc = we - wb;
    p->key = derive_key(c->seed, kPermTag);
    Part tmp = p->part;
    p->A = (uint64_t)tmp.E * (tmp.prefix_len(we) - tmp.prefix_len(wb));
    if (p->A >= 0xFFFFFFFFull) {
        delete p;
        return fail(CLAIRPLAN_EOVERFLOW, "more than 2^32-1 stream entries in one handle; shard the "
                                         "workers over several handles");
    }
    if (cudaStreamCreateWithFlags(&p->stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreate(&p->ev0) != cudaSuccess || cudaEventCreate(&p->ev1) != cudaSuccess) {
        delete p;
        return fail(CLAIRPLAN_ECUDA, "stream/event creation failed");
    }
    for (auto& e : p->sev) cudaEventCreate(&e);
    if (!p->sizes.ensure((size_t)c->samples * sizeof(double))) {
        delete p;
        return fail(CLAIRPLAN_ENOMEM, "device allocation failed (sizes)");
    }
    cudaError_t e = cudaSuccess;
    if (c->sizes_mb)
        // on the handle's (non-blocking) stream: every kernel reading the sizes runs there
        e = cudaMemcpyAsync(p->sizes.get<double>(), c->sizes_mb, (size_t)c->samples * 8,
                            c->sizes_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                            p->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(p->stream);  // the caller may free sizes_mb
    if (e != cudaSuccess) {
        delete p;
        return fail(CLAIRPLAN_ECUDA, std::string("sizes upload: ") + cudaGetErrorString(e));
    }
    *out = p;
    return 0;
}

int clairplan_destroy(clairplan_t p) {
    if (!p) return 0;
    cudaSetDevice(p->device);
    delete p;
    return 0;
}

int clairplan_build(clairplan_t p) {
    if (!p) return fail(CLAIRPLAN_EINVAL, "null plan");
    if (p->generic) return fail(CLAIRPLAN_EINVAL, "plan was created from explicit streams");
    CK(cudaSetDevice(p->device));
    p->built = false;
    p->v2 = false;
    const char* force = path_switch("CLAIRPLAN_FORCE_V1");
    if (v2_ok(p) && !(force && force[0] == '1')) return build_seed_path_v2(p, nullptr);
    return build_seed_path(p);
}

int clairplan_build_export(clairplan_t p, const double* host_sizes, uint32_t* streams_out,
                           uint64_t streams_cap, uint32_t* class_lists_out, uint64_t cl_cap,
                           uint64_t* offsets_out, uint32_t* holders_out, uint64_t holders_cap) {
    if (!p || !streams_out || !offsets_out) return fail(CLAIRPLAN_EINVAL, "null argument");
    if (p->generic) return fail(CLAIRPLAN_EINVAL, "plan was created from explicit streams");
    CK(cudaSetDevice(p->device));
    if (streams_cap < p->part.E * (p->part.prefix_len(p->part.wend) - p->part.prefix_len(p->part.wbegin)))
        return fail(CLAIRPLAN_ERANGE, "stream buffer too small");
    if (!p->xstream) {
        CK(cudaStreamCreateWithFlags(&p->xstream, cudaStreamNonBlocking));
        CK(cudaEventCreateWithFlags(&p->xev, cudaEventDisableTiming));
    }
    if (host_sizes)
        if (int rc = clairplan_set_sizes(p, host_sizes, 0)) return rc;
    p->x_streams = streams_out;
    p->x_class = class_lists_out;
    p->x_class_cap = class_lists_out ? cl_cap : 0;
    p->x_class_done = false;
    int rc = clairplan_build(p);
    const bool copied = p->v2;  // the v2 build issued the stream copy on xstream
    bool cl_copied = p->x_class_done;  // ... and the class lists
    p->x_streams = nullptr;
    p->x_class = nullptr;
    if (rc) {
        cudaStreamSynchronize(p->xstream);
        return rc;
    }
    // output capacities are checked before any further copy is issued; an error after the
    // build waits for the stream copy already in flight on xstream (the caller may free or
    // reuse its buffers as soon as this returns)
    uint64_t cl_need = 0;
    for (uint32_t w = 0; w < p->nloc; ++w)
        for (uint32_t j = 0; j < p->cfg.num_classes; ++j)
            cl_need += p->class_len_h[(size_t)w * (p->cfg.num_classes + 1) + j];
    if (cl_cap < cl_need || holders_cap < p->H || (cl_need && !class_lists_out) ||
        (p->H && !holders_out)) {
        cudaStreamSynchronize(p->xstream);
        cudaStreamSynchronize(p->stream);
        return fail(CLAIRPLAN_ERANGE, cl_cap < cl_need || holders_cap < p->H
                                          ? "output buffer too small"
                                          : "null output buffer");
    }
    if (!copied)
        CK(cudaMemcpyAsync(streams_out, p->stream_buf.get<uint32_t>(), p->A * 4, cudaMemcpyDeviceToHost,
                           p->stream));
    if (cl_copied && p->H != p->D) {  // (not expected: every candidate was cached) exact copy
        CK(cudaStreamSynchronize(p->xstream));
        cl_copied = false;
    }
    if (!cl_copied)
        if (int rc2 = clairplan_export_class_lists_async(p, class_lists_out, cl_cap)) {
            cudaStreamSynchronize(p->xstream);
            cudaStreamSynchronize(p->stream);
            return rc2;
        }
    CK(cudaMemcpyAsync(offsets_out, p->holder_off_dev, ((uint64_t)p->part.F + 1) * 8,
                       cudaMemcpyDeviceToHost, p->stream));
    if (p->H) CK(cudaMemcpyAsync(holders_out, p->holders_dev, p->H * 12, cudaMemcpyDeviceToHost, p->stream));
    CK(cudaStreamSynchronize(p->stream));
    CK(cudaStreamSynchronize(p->xstream));
    return 0;
}

int clairplan_stats_get(clairplan_t p, clairplan_stats* s) {
    if (!p || !s) return fail(CLAIRPLAN_EINVAL, "null argument");
    s->accesses = p->A;
    s->pairs = p->D;
    s->holders = p->H;
    s->rejections = p->rejections;
    s->device_ms = p->device_ms;
    s->path = !p->v2 ? CLAIRPLAN_PATH_V1 : p->allfit ? CLAIRPLAN_PATH_ALLFIT : CLAIRPLAN_PATH_TIER;
    s->reserved = 0;
    return 0;
}

uint64_t clairplan_launch_count(clairplan_t p) { return p ? p->launches : 0; }

int clairplan_device_streams(clairplan_t p, const uint32_t** entries, uint64_t* total) {
    if (!p || !p->built) return fail(CLAIRPLAN_EINVAL, "plan not built");
    *entries = p->stream_buf.get<uint32_t>();
    *total = p->A;
    return 0;
}

uint64_t clairplan_stream_offset(clairplan_t p, uint32_t w) {
    if (!p) return 0;
    if (w < p->part.wbegin) w = p->part.wbegin;
    if (w > p->part.wend) w = p->part.wend;
    return p->part.stream_offset(w);
}

int clairplan_class_list_bounds(clairplan_t p, uint64_t* off, uint64_t* len) {
    if (!p || !p->built) return fail(CLAIRPLAN_EINVAL, "plan not built");
    const uint32_t J = p->cfg.num_classes;
    for (uint32_t w = 0; w < p->nloc; ++w)
        for (uint32_t j = 0; j < J; ++j) {
            off[(size_t)w * J + j] = p->class_start_h[(size_t)w * (J + 1) + j];
            len[(size_t)w * J + j] = p->class_len_h[(size_t)w * (J + 1) + j];
        }
    return 0;
}

int clairplan_device_class_lists(clairplan_t p, const uint32_t** entries) {
    if (!p || !p->built) return fail(CLAIRPLAN_EINVAL, "plan not built");
    *entries = p->class_entries.get<uint32_t>();
    return 0;
}

int clairplan_device_holders(clairplan_t p, const uint64_t** offsets, const uint32_t** holders,
                             uint64_t* count) {
    if (!p || !p->built) return fail(CLAIRPLAN_EINVAL, "plan not built");
    *offsets = p->holder_off_dev;
    *holders = p->holders_dev;
    *count = p->H;
    return 0;
}

int clairplan_export_stream(clairplan_t p, uint32_t w, uint32_t* out, uint64_t cap, uint64_t* len) {
    if (!p || !p->built) return fail(CLAIRPLAN_EINVAL, "plan not built");
    if (w < p->part.wbegin || w >= p->part.wend) return fail(CLAIRPLAN_EINVAL, "worker not in plan");
    const uint64_t a = p->part.stream_offset(w), b = p->part.stream_offset(w + 1);
    *len = b - a;
    if (cap < b - a) return fail(CLAIRPLAN_ERANGE, "output buffer too small");
    CK(cudaSetDevice(p->device));
    CK(cudaMemcpy(out, p->stream_buf.get<uint32_t>() + a, (b - a) * 4, cudaMemcpyDeviceToHost));
    return 0;
}

int clairplan_export_streams(clairplan_t p, uint32_t* out, uint64_t cap) {
    if (!p || !p->built) return fail(CLAIRPLAN_EINVAL, "plan not built");
    if (cap < p->A) return fail(CLAIRPLAN_ERANGE, "output buffer too small");
    CK(cudaSetDevice(p->device));
    CK(cudaMemcpy(out, p->stream_buf.get<uint32_t>(), p->A * 4, cudaMemcpyDeviceToHost));
    return 0;
}

}  // extern "C"

namespace clairplan {
// class lists back to back in (worker, class) order, on the handle's stream
int clairplan_export_class_lists_async(clairplan_t p, uint32_t* out, uint64_t cap) {
    const uint32_t J = p->cfg.num_classes;
    uint64_t need_n = 0;
    for (uint32_t w = 0; w < p->nloc; ++w)
        for (uint32_t j = 0; j < J; ++j) need_n += p->class_len_h[(size_t)w * (J + 1) + j];
    if (cap < need_n) return fail(CLAIRPLAN_ERANGE, "output buffer too small");
    if (need_n == 0) return 0;
    if (!out) return fail(CLAIRPLAN_EINVAL, "null class-list buffer");
    if (p->v2 && p->cl_contig) {
        CK(cudaMemcpyAsync(out, p->class_entries.get<uint32_t>(), need_n * 4, cudaMemcpyDeviceToHost,
                           p->stream));
        return 0;
    }
    uint64_t o = 0;
    for (uint32_t w = 0; w < p->nloc; ++w) {
        const uint64_t a = p->class_start_h[(size_t)w * (J + 1)];
        uint64_t n = 0;
        for (uint32_t j = 0; j < J; ++j) n += p->class_len_h[(size_t)w * (J + 1) + j];
        if (n)
            CK(cudaMemcpyAsync(out + o, p->class_entries.get<uint32_t>() + a, n * 4,
                               cudaMemcpyDeviceToHost, p->stream));
        o += n;
    }
    return 0;
}
}  // namespace clairplan

extern "C" {

int clairplan_export_class_lists(clairplan_t p, uint32_t* out, uint64_t cap) {
    if (!p || !p->built) return fail(CLAIRPLAN_EINVAL, "plan not built");
    const uint32_t J = p->cfg.num_classes;
    uint64_t need_n = 0;
    for (uint32_t w = 0; w < p->nloc; ++w)
        for (uint32_t j = 0; j < J; ++j) need_n += p->class_len_h[(size_t)w * (J + 1) + j];
    if (cap < need_n) return fail(CLAIRPLAN_ERANGE, "output buffer too small");
    if (need_n == 0) return 0;
    CK(cudaSetDevice(p->device));
    if (p->v2 && p->cl_contig) {  // class lists are stored back to back in (worker, class) order
        CK(cudaMemcpy(out, p->class_entries.get<uint32_t>(), need_n * 4, cudaMemcpyDeviceToHost));
        return 0;
    }
    uint64_t o = 0;
    for (uint32_t w = 0; w < p->nloc; ++w) {
        // classes 1..J of a worker are adjacent in the class-partitioned array
        const uint64_t a = p->class_start_h[(size_t)w * (J + 1)];
        uint64_t n = 0;
        for (uint32_t j = 0; j < J; ++j) n += p->class_len_h[(size_t)w * (J + 1) + j];
        if (n) CK(cudaMemcpy(out + o, p->class_entries.get<uint32_t>() + a, n * 4, cudaMemcpyDeviceToHost));
        o += n;
    }
    return 0;
}

int clairplan_export_holders(clairplan_t p, uint64_t* offsets, uint32_t* holders, uint64_t cap) {
    if (!p || !p->built) return fail(CLAIRPLAN_EINVAL, "plan not built");
    if (cap < p->H) return fail(CLAIRPLAN_ERANGE, "output buffer too small");
    CK(cudaSetDevice(p->device));
    CK(cudaMemcpy(offsets, p->holder_off_dev, ((uint64_t)p->part.F + 1) * 8, cudaMemcpyDeviceToHost));
    if (p->H) CK(cudaMemcpy(holders, p->holders_dev, p->H * 12, cudaMemcpyDeviceToHost));
    return 0;
}

int clairplan_export_counts(clairplan_t p, uint32_t w, uint32_t* counts) {
    if (!p || !p->built) return fail(CLAIRPLAN_EINVAL, "plan not built");
    if (w < p->part.wbegin || w >= p->part.wend) return fail(CLAIRPLAN_EINVAL, "worker not in plan");
    if (p->generic) return fail(CLAIRPLAN_EINVAL, "counts of an explicit-stream plan are the caller's");
    CK(cudaSetDevice(p->device));
    const uint64_t a = p->part.stream_offset(w), b = p->part.stream_offset(w + 1);
    DevBuf tmp;
    if (!tmp.ensure((size_t)p->part.F * 4)) return fail(CLAIRPLAN_ENOMEM, "device allocation failed");
    CK(cudaMemsetAsync(tmp.p, 0, (size_t)p->part.F * 4, p->stream));
    if (b > a) launch_stream_hist(p->stream, p->stream_buf.get<uint32_t>() + a, b - a, tmp.get<uint32_t>());
    CK(cudaStreamSynchronize(p->stream));
    CK(cudaGetLastError());
    CK(cudaMemcpy(counts, tmp.p, (size_t)p->part.F * 4, cudaMemcpyDeviceToHost));
    return 0;
}

int clairplan_epoch_permutation(uint64_t seed, uint32_t epoch, uint32_t samples, uint32_t* out,
                                int device) {
    if (samples < 1) return fail(CLAIRPLAN_EINVAL, "permutation needs samples >= 1");  // access.cpp:53
    if (int rc = check_device(device)) return rc;
    clairplan_plan p;
    p.device = device;
    CK(cudaStreamCreateWithFlags(&p.stream, cudaStreamNonBlocking));
    p.part = make_part(samples, 1, 1, 1, true, 0, 1);
    p.key = derive_key(seed, kPermTag);
    p.rej_ebase = epoch;
    if (int rc = alloc_rej(&p, 1)) return rc;
    DevBuf perm;
    if (!perm.ensure((size_t)samples * 4)) return fail(CLAIRPLAN_ENOMEM, "device allocation failed");
    for (int attempt = 0; attempt < 3; ++attempt) {
        if (int rc = enqueue_perms(&p, nullptr, nullptr, perm.get<uint32_t>(), epoch, 1)) return rc;
        std::vector<uint32_t> flags(1, 0);
        CK(cudaMemcpyAsync(&flags[0], p.rej_flag.get<uint32_t>(), 4,
                           cudaMemcpyDeviceToHost, p.stream));
        CK(cudaStreamSynchronize(p.stream));
        bool any = false;
        if (int rc = resolve_rejections(&p, flags, &any)) return rc;
        if (any) continue;
        CK(cudaMemcpy(out, perm.p, (size_t)samples * 4, cudaMemcpyDeviceToHost));
        return 0;
    }
    return fail(CLAIRPLAN_ECUDA, "rejection tables did not converge");
}

static const char* kStageNames[clairplan_plan::kStages] = {
    "permutations+streams", "sample_histogram", "candidate_count", "candidate_write",
    "tier_order", "first_fit", "class_lists", "holder_csr"};

const char* clairplan_stage_name(uint32_t i) {
    return i < (uint32_t)clairplan_plan::kStages ? kStageNames[i] : "";
}

int clairplan_stage_times(clairplan_t p, double* ms, uint32_t n) {
    if (!p || !p->built) return fail(CLAIRPLAN_EINVAL, "plan not built");
    for (uint32_t i = 0; i < n && i < (uint32_t)clairplan_plan::kStages; ++i) ms[i] = p->stage_ms[i];
    return clairplan_plan::kStages;
}

int clairplan_set_sizes(clairplan_t p, const double* sizes_mb, int on_device) {
    if (!p || !sizes_mb) return fail(CLAIRPLAN_EINVAL, "null argument");
    CK(cudaSetDevice(p->device));
    if (!p->sizes.ensure((size_t)p->part.F * 8)) return fail(CLAIRPLAN_ENOMEM, "device allocation failed");
    CK(cudaMemcpyAsync(p->sizes.get<double>(), sizes_mb, (size_t)p->part.F * 8,
                       on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, p->stream));
    return 0;
}

// ---- multi-GPU building blocks ---------------------------------------------------------
int clairplan_generate_perms(clairplan_t p, uint32_t epoch_begin, uint32_t epoch_count,
                             uint32_t* d_out) {
    if (!p || p->generic) return fail(CLAIRPLAN_EINVAL, "invalid plan");
    if (epoch_count == 0) return 0;
    if (epoch_begin + epoch_count > p->part.E) return fail(CLAIRPLAN_EINVAL, "epoch range outside plan");
    CK(cudaSetDevice(p->device));
    if (int rc = alloc_rej(p, p->part.E)) return rc;
    for (int attempt = 0; attempt < 3; ++attempt) {
        p->launches = 0;
        if (int rc = enqueue_perms(p, nullptr, nullptr, d_out, epoch_begin, epoch_count)) return rc;
        std::vector<uint32_t> flags(p->part.E);
        CK(cudaMemcpyAsync(flags.data(), p->rej_flag.get<uint32_t>(), flags.size() * 4,
                           cudaMemcpyDeviceToHost, p->stream));
        CK(cudaStreamSynchronize(p->stream));
        bool any = false;
        if (int rc = resolve_rejections(p, flags, &any)) return rc;
        if (!any) return 0;
    }
    return fail(CLAIRPLAN_ECUDA, "rejection tables did not converge");
}

int clairplan_epoch_prefix(clairplan_t p, uint32_t worker, uint64_t* entries) {
    if (!p || !entries) return fail(CLAIRPLAN_EINVAL, "null argument");
    if (worker > p->part.N) return fail(CLAIRPLAN_EINVAL, "worker out of range");
    *entries = p->part.prefix_len(worker);
    return 0;
}

static int generate_streams_impl(clairplan_plan* p, uint32_t epoch_begin, uint32_t epoch_count,
                                 uint32_t* d_out, const StreamDst* dst) {
    if (!p || p->generic) return fail(CLAIRPLAN_EINVAL, "invalid plan");
    if (epoch_count == 0) return 0;
    if (!d_out && !(dst && dst->G)) return fail(CLAIRPLAN_EINVAL, "null output");
    if (epoch_begin + epoch_count > p->part.E) return fail(CLAIRPLAN_EINVAL, "epoch range outside plan");
    CK(cudaSetDevice(p->device));
    const Part& pp = p->part;
    if ((uint64_t)epoch_count * pp.P >= (1ull << 32))
        return fail(CLAIRPLAN_EOVERFLOW, "epoch range holds 2^32 or more stream entries");
    Part sp = make_part(pp.F, pp.N, pp.B, epoch_count, pp.drop_last != 0, 0, pp.N);
    sp.ebase = epoch_begin;
    if (int rc = alloc_rej(p, p->part.E)) return rc;
    // a dense sharded build follows: the shuffle writes this range's whole inverse rows into
    // the handle's inv (CLAIRPLAN_OWN_INV=0 disables, A/B)
    p->inv_own_lo = p->inv_own_hi = 0;
    uint32_t* own_inv = nullptr;
    static const bool own_ok = ab_knob("CLAIRPLAN_OWN_INV", 1) != 0;
    if (own_ok && v2_ok(p) && !sharded_sparse(p)) {
        bool ok = true;
        own_inv = need<uint32_t>(p->inv, (uint64_t)pp.E * pp.Fp, ok);
        if (!ok) own_inv = nullptr;
    }
    for (int attempt = 0; attempt < 3; ++attempt) {
        p->launches = 0;
        CK(cudaEventRecord(p->ev0, p->stream));
        if (int rc = enqueue_perms(p, d_out, own_inv, nullptr, epoch_begin, epoch_count, &sp, dst)) return rc;
        std::vector<uint32_t> flags(p->part.E);
        CK(cudaMemcpyAsync(flags.data(), p->rej_flag.get<uint32_t>(), flags.size() * 4,
                           cudaMemcpyDeviceToHost, p->stream));
        CK(cudaEventRecord(p->ev1, p->stream));
        CK(cudaStreamSynchronize(p->stream));
        bool any = false;
        if (int rc = resolve_rejections(p, flags, &any)) return rc;
        if (!any) {
            float ms = 0;
            CK(cudaEventElapsedTime(&ms, p->ev0, p->ev1));
            p->gen_ms = ms;
            if (own_inv) {
                p->inv_own_lo = epoch_begin;
                p->inv_own_hi = epoch_begin + epoch_count;
            }
            return 0;
        }
    }
    return fail(CLAIRPLAN_ECUDA, "rejection tables did not converge");
}

int clairplan_generate_streams(clairplan_t p, uint32_t epoch_begin, uint32_t epoch_count,
                               uint32_t* d_out) {
    return generate_streams_impl(p, epoch_begin, epoch_count, d_out, nullptr);
}

int clairplan_generate_streams_p2p(clairplan_t p, uint32_t epoch_begin, uint32_t epoch_count,
                                   const uint64_t* dst_base, const int64_t* dst_delta,
                                   const uint32_t* worker_bounds, uint32_t nranks) {
    if (!p || !dst_base || !dst_delta || !worker_bounds) return fail(CLAIRPLAN_EINVAL, "invalid argument");
    if (nranks < 1 || nranks > kMaxPeers) return fail(CLAIRPLAN_EINVAL, "1..16 ranks supported");
    if (worker_bounds[0] != 0 || worker_bounds[nranks] != p->part.N)
        return fail(CLAIRPLAN_EINVAL, "worker bounds must cover [0, workers)");
    StreamDst d{};
    d.G = nranks;
    for (uint32_t r = 0; r <= nranks; ++r) d.wb[r] = worker_bounds[r];
    for (uint32_t r = 0; r < nranks; ++r) {
        if (!dst_base[r]) return fail(CLAIRPLAN_EINVAL, "null destination buffer");
        d.base[r] = reinterpret_cast<uint32_t*>(dst_base[r]);
        d.delta[r] = (long long)dst_delta[r];
    }
    FycDev fg;
    if (!fyc_ready(p, p->part.F, fg))
        return fail(CLAIRPLAN_EINVAL, "peer-memory stream writes need the bucketed shuffle");
    return generate_streams_impl(p, epoch_begin, epoch_count, nullptr, &d);
}

int clairplan_p2p_supported(clairplan_t p) {
    FycDev fg;
    return (p && !p->generic && !path_switch("CLAIRPLAN_FY_LISTS") && fyc_ready(p, p->part.F, fg)) ? 1 : 0;
}

int clairplan_recv_buffer(clairplan_t p, uint32_t i, void** d_ptr, void* ipc_handle) {
    if (!p || !d_ptr || i >= 4) return fail(CLAIRPLAN_EINVAL, "invalid argument");
    CK(cudaSetDevice(p->device));
    if (p->recvbufs.size() <= i) p->recvbufs.resize(i + 1, nullptr);
    if (!p->recvbufs[i]) {
        void* b = nullptr;
        if (cudaMalloc(&b, std::max<uint64_t>(p->A, 1) * 4) != cudaSuccess) {
            cudaGetLastError();
            return fail(CLAIRPLAN_ENOMEM, "receive buffer allocation failed");
        }
        p->recvbufs[i] = b;
    }
    *d_ptr = p->recvbufs[i];
    if (ipc_handle) {
        cudaIpcMemHandle_t h;
        CK(cudaIpcGetMemHandle(&h, p->recvbufs[i]));
        memcpy(ipc_handle, &h, sizeof(h));
    }
    return 0;
}

int clairplan_open_peer_buffer(clairplan_t p, const void* ipc_handle, void** d_ptr) {
    if (!p || !ipc_handle || !d_ptr) return fail(CLAIRPLAN_EINVAL, "invalid argument");
    CK(cudaSetDevice(p->device));
    cudaIpcMemHandle_t h;
    memcpy(&h, ipc_handle, sizeof(h));
    void* ptr = nullptr;
    CK(cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess));
    p->peerbufs.push_back(ptr);
    *d_ptr = ptr;
    return 0;
}

int clairplan_build_from_streams(clairplan_t p, const uint32_t* d_recv,
                                 const uint32_t* epoch_bounds, uint32_t nsrc) {
    if (!p || p->generic || !d_recv || !epoch_bounds) return fail(CLAIRPLAN_EINVAL, "invalid argument");
    if (nsrc < 1 || nsrc > kMaxRanks) return fail(CLAIRPLAN_EINVAL, "1..64 source ranks supported");
    if (epoch_bounds[0] != 0 || epoch_bounds[nsrc] != p->part.E)
        return fail(CLAIRPLAN_EINVAL, "epoch bounds must cover [0, epochs)");
    EpochSplit es{};
    es.G = nsrc;
    for (uint32_t r = 0; r <= nsrc; ++r) {
        es.eb[r] = epoch_bounds[r];
        if (r && es.eb[r] < es.eb[r - 1]) return fail(CLAIRPLAN_EINVAL, "epoch bounds must ascend");
    }
    CK(cudaSetDevice(p->device));
    if (!v2_ok(p)) return fail(CLAIRPLAN_EINVAL, "configuration not supported by the sharded path");
    p->built = false;
    p->v2 = false;
    const int rc = build_seed_path_v2(p, nullptr, d_recv, &es);
    p->inv_own_lo = p->inv_own_hi = 0;  // the rows are the build's now (reassign, later builds)
    return rc;
}

int clairplan_build_from_perms(clairplan_t p, const uint32_t* d_perms) {
    if (!p || p->generic || !d_perms) return fail(CLAIRPLAN_EINVAL, "invalid argument");
    CK(cudaSetDevice(p->device));
    if (!v2_ok(p)) return fail(CLAIRPLAN_EINVAL, "configuration not supported by the sharded path");
    p->built = false;
    p->v2 = false;
    return build_seed_path_v2(p, d_perms);
}

int clairplan_set_counts_hook(clairplan_t p, uint32_t* d_counts, void* stream,
                              void (*fn)(void*), void* user) {
    if (!p) return fail(CLAIRPLAN_EINVAL, "null plan");
    if (fn && !d_counts) return fail(CLAIRPLAN_EINVAL, "counts hook needs a device buffer");
    p->hook_counts = d_counts;
    p->hook_stream = (cudaStream_t)stream;
    p->hook_fn = fn;
    p->hook_user = user;
    p->hook_fired = false;
    return 0;
}

int clairplan_counts_hook_valid(clairplan_t p) {
    return (p && p->built && p->hook_fired && p->allfit && p->H == p->D) ? 1 : 0;
}

int clairplan_holder_counts(clairplan_t p, uint32_t* d_out) {
    if (!p || !p->built || p->generic) return fail(CLAIRPLAN_EINVAL, "plan not built");
    CK(cudaSetDevice(p->device));
    const uint32_t F = p->part.F;
    const uint32_t* src = (p->H == p->D) ? p->pair_count.get<uint32_t>() : p->hcount.get<uint32_t>();
    if (p->cfg.num_classes == 0) CK(cudaMemsetAsync(d_out, 0, (size_t)F * 4, p->stream));
    else CK(cudaMemcpyAsync(d_out, src, (size_t)F * 4, cudaMemcpyDeviceToDevice, p->stream));
    CK(cudaStreamSynchronize(p->stream));
    return 0;
}

// Re-planning for capacity sweeps: same streams and tier order, new
// capacities -> rerun only first fit, class lists and holders (the reference rebuilds the
// whole assignment per grid point, simulator.cpp:457-465 -> policies.cpp:449-454).
int clairplan_reassign(clairplan_t p, const double* capacities_mb) {
    if (!p || !p->built || p->generic) return fail(CLAIRPLAN_EINVAL, "plan not built");
    if (!p->v2) return fail(CLAIRPLAN_EINVAL, "re-planning needs the v2 device path");
    if (p->cfg.num_classes && !capacities_mb) return fail(CLAIRPLAN_EINVAL, "null capacities");
    CK(cudaSetDevice(p->device));
    p->caps.assign(capacities_mb, capacities_mb + p->cfg.num_classes);
    p->ws.used = 0;
    p->launches = 0;
    CK(cudaEventRecord(p->ev0, p->stream));
    if (!p->tier_ready)  // the build took the all-fit path: materialise the tier order once
        if (int rc = tier_order_v2(p)) return rc;
    p->allfit = false;
    if (int rc = assign_v2(p)) return rc;
    CK(cudaEventRecord(p->ev1, p->stream));
    CK(cudaEventSynchronize(p->ev1));
    CK(cudaGetLastError());
    if (p->ws.overflow) return fail(CLAIRPLAN_ENOMEM, "internal workspace overflow");
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, p->ev0, p->ev1));
    p->device_ms = ms;
    return 0;
}

}  // extern "C"
