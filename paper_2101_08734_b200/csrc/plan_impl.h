// Private host-side declarations of the clairplan handle (plan.cu, generic.cu).
#pragma once
#include <cuda_runtime.h>
#include <stdio.h>
#include <string.h>

#include <stdlib.h>

#include <algorithm>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/clairplan.h"
#include "internal.h"

namespace clairplan {

extern thread_local std::string g_err;

inline int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

#define CK(call)                                                                      \
    do {                                                                              \
        cudaError_t e_ = (call);                                                      \
        if (e_ != cudaSuccess)                                                        \
            return fail(CLAIRPLAN_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
    } while (0)

struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    ~DevBuf() {
        if (p) cudaFree(p);
    }
    template <typename T>
    T* get() const { return static_cast<T*>(p); }
    // grow-only; returns false on allocation failure
    bool ensure(size_t need) {
        if (need <= bytes) return true;
        if (p) cudaFree(p);
        p = nullptr;
        bytes = 0;
        size_t b = need + (need >> 3) + 256;
        if (cudaMalloc(&p, b) != cudaSuccess) {
            cudaGetLastError();
            p = nullptr;
            return false;
        }
        bytes = b;
        return true;
    }
};

constexpr uint32_t kRejCap = 16;

inline int check_device(int device) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
        cudaGetLastError();
        return fail(CLAIRPLAN_ENODEV, "no CUDA device available (clairplan has no CPU fallback)");
    }
    if (device < 0 || device >= n) return fail(CLAIRPLAN_ENODEV, "CUDA device ordinal out of range");
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10)
        return fail(CLAIRPLAN_ENODEV, "clairplan kernels are built for sm_100a (B200) only");
    CK(cudaSetDevice(device));
    return 0;
}

inline int validate_partition(uint64_t F, uint32_t N, uint32_t B, uint32_t E) {
    // access.cpp:41-50, same messages
    if (F < 1) return fail(CLAIRPLAN_EINVAL, "dataset must have at least one sample");
    if (N < 1) return fail(CLAIRPLAN_EINVAL, "num_workers must be >= 1");
    if (E < 1) return fail(CLAIRPLAN_EINVAL, "epochs must be >= 1");
    if (B < N) return fail(CLAIRPLAN_EINVAL, "global batch must be >= num_workers");
    if (B > F)
        return fail(CLAIRPLAN_EINVAL, "global batch " + std::to_string(B) +
                                          " exceeds dataset size " + std::to_string(F));
    return 0;
}

}  // namespace clairplan

using namespace clairplan;

struct clairplan_plan {
    int device = 0;
    cudaStream_t stream = nullptr;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    static constexpr int kStages = 8;
    cudaEvent_t sev[kStages + 1] = {};  // stage boundaries of the last build
    double stage_ms[kStages] = {};
    clairplan_config cfg{};
    std::vector<double> caps;
    Part part{};
    uint32_t nloc = 0;
    uint64_t key = 0;
    uint64_t A = 0, D = 0, H = 0, rejections = 0;
    double device_ms = 0;
    double gen_ms = 0;               // device time of the last clairplan_generate_streams
    bool built = false;
    bool generic = false;
    uint64_t launches = 0;
    uint32_t rej_ebase = 0;  // rejection tables are indexed by epoch - rej_ebase

    DevBuf sizes, stream_buf, info, pair_count, pair_off, segcnt, seg_off, wbeg, wlen;
    DevBuf cand_k, cand_info, cand_cls, order, sorted_size;
    DevBuf keys, vals, okeys, ovals, taken, seqsz, dest;
    DevBuf class_entries, class_start, class_len, holders, holders_tmp, hcount, hoff;
    DevBuf head, next, q, scratch, counters, rej_flag, rej_step, rej_cum, rej_count;
    DevBuf wsbuf;
    DevBuf cand_w, dfirst, dcounts;  // explicit-stream (generic) path
    DevBuf inv, info16, rank16, cbase, seghist, sorted_base, blkmask, blkbase, planes, ccount, cpre;
    DevBuf wsum, wcnt, chstatus, allfit_gate;  // all-fit: worker sums / counts, look-back, decision
    bool cl_contig = true;           // class lists back to back (tier path) or at stream offsets
    DevBuf koff, sp_cur, csr, cpos, soff, einfo, erank;  // sparse sample-major passes (sharded)
    // contiguous-bucket shuffle (perm_fyc.cu): host geometry of the handle's F, its device
    // copy (block starts, capacities, target cells, region offsets), bucket regions, cursors
    FycHost fych;
    DevBuf fyc_geo, fyc_region, fyc_cursor;
    bool fyc_off = false;            // a block region overflowed once: linked-list path
    DevBuf merge_buf;                // clairplan_merge_holder_counts scratch (own: may overlap a build)
    DevBuf sorted_k;                 // tier path: sample id of every tier position (seg_write3)
    bool ssize_pending = false;      // sorted_size not yet gathered (class 1's ff_stats does it)
    DevBuf sched;                    // in-order work claim counters (seg_write3, hp_fill)
    DevBuf hpos;                     // tier path: [E][Fp] class << 28 | class-list position (hp_fill)
    bool hp_path = false;            // last assignment wrote hpos (holder_hp replaces holder_tile)
    bool info8 = false;              // info rows of the last dense build are u8 (else u16)
    // whole-worker candidate size sums of the last seed build (sample pass; all-fit test) on
    // the host: a class whose capacity holds every worker's total takes all its remaining
    // candidates (first_fit_classes)
    std::vector<unsigned long long> wsum_h;
    std::vector<uint32_t> wcnt_h;
    bool sums_ok = false;
    bool sparse = false;             // last build used the sparse passes
    bool allfit = false;             // last build took the all-fit path (no tier order)
    bool tier_ready = false;         // dest / sorted_size / block masks hold the tier order
    bool hist_ready = false;         // seghist / sorted_base hold the count histograms
    bool v2 = false;                 // fast seed path in use for the last build
    uint32_t v2_mb = 0;              // blocks per segment / total blocks of the last v2 build
    uint64_t v2_nblk = 0;
    uint32_t maxcount = 0;           // generic path: largest frequency value
    Workspace ws;

    std::vector<uint64_t> class_start_h, class_len_h;  // [(w, d)] d in 0..J
    std::vector<uint32_t> rej_step_h, rej_cum_h, rej_count_h;
    const uint64_t* holder_off_dev = nullptr;
    const uint32_t* holders_dev = nullptr;

    cudaStream_t xstream = nullptr;   // build_export: stream of the overlapped output copy
    cudaEvent_t xev = nullptr;
    uint32_t* x_streams = nullptr;     // build_export: host stream buffer of the running build
    uint32_t* x_class = nullptr;       // build_export: host class-list buffer and its capacity
    uint64_t x_class_cap = 0;
    bool x_class_done = false;         // the class lists were copied during the build (xstream)
    bool h_known = false;              // first fit: every candidate assigned (H = D) known on host
    // counts hook (multi-GPU holder-offset merge overlapped with the build's tail): once the
    // per-sample pair counts exist, they are copied to hook_counts, hook_stream waits for them
    // and hook_fn runs on the host (it enqueues the all-gather); valid if the build then took
    // the all-fit path (holder counts = pair counts) without a rejection rerun
    void* hook_counts = nullptr;
    cudaStream_t hook_stream = nullptr;
    void (*hook_fn)(void*) = nullptr;
    void* hook_user = nullptr;
    cudaEvent_t hook_ev = nullptr;
    bool hook_fired = false;
    // epochs whose whole inverse rows clairplan_generate_streams left in inv (dense sharded
    // build: not rebuilt from the received streams); [0, 0) = none
    uint32_t inv_own_lo = 0, inv_own_hi = 0;
    std::vector<void*> recvbufs;   // multi-GPU fused exchange: this rank's receive buffers
    std::vector<void*> peerbufs;   // opened peers' receive buffers (CUDA IPC)
    ~clairplan_plan() {
        for (void* b : peerbufs) cudaIpcCloseMemHandle(b);
        for (void* b : recvbufs)
            if (b) cudaFree(b);
        if (hook_ev) cudaEventDestroy(hook_ev);
        if (xstream) cudaStreamDestroy(xstream);
        if (xev) cudaEventDestroy(xev);
        if (stream) cudaStreamDestroy(stream);
        if (ev0) cudaEventDestroy(ev0);
        if (ev1) cudaEventDestroy(ev1);
        for (auto& e : sev)
            if (e) cudaEventDestroy(e);
    }
    void mark(int i) {
        if (sev[i]) cudaEventRecord(sev[i], stream);
        static const bool dbg = [] {
            return ab_flag("CLAIRPLAN_DEBUG_SYNC");
        }();
        if (dbg) {
            const cudaError_t err = cudaStreamSynchronize(stream);
            if (err != cudaSuccess) {
                fprintf(stderr, "clairplan: CUDA error before stage mark %d: %s\n", i,
                        cudaGetErrorString(err));
                abort();
            }
        }
    }
};


namespace clairplan {
template <typename T>
inline T* need(DevBuf& b, uint64_t n, bool& ok) {
    if (!b.ensure(std::max<uint64_t>(n, 1) * sizeof(T))) ok = false;
    return b.get<T>();
}


int assign_tiers(clairplan_plan* p);
int generic_holders(clairplan_plan* p);
void launch_generic_count_keys(cudaStream_t s, const uint32_t* cnt, uint64_t n, uint32_t maxc,
                               uint32_t* keys);
int ensure_ws(clairplan_plan* p, uint64_t n_elems, uint32_t nseg);
int clairplan_export_class_lists_async(clairplan_t p, uint32_t* out, uint64_t cap);
}  // namespace clairplan
