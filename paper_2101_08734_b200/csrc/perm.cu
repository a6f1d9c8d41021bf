// K1-K3, linked-list resolution: the fallback of perm_fyc.cu (a bucket region overflow, or
// a geometry that does not apply).  Bit-exact parallel Fisher-Yates (rng.cpp:15-24,
// access.cpp:52-57) fused with the partition into per-worker streams (access.cpp:14-39, 59-78).
//
// The sequential shuffle "for i = F-1 .. 1: swap(a[i], a[j_i])" is resolved without
// executing the swaps in order.  Group the steps by target: writers of y are the steps
// i >= y with j_i = y, ascending w_1 < ... < w_m.
//   q(y)   = smallest writer of y other than y itself (the last write into y before step y)
//   succ(i)= next larger writer of the same target (the last write into j_i before step i)
//   V(x)   = value at position x just before step x = V(q(x)) if q(x) exists, else x
//   out[i] = V(succ(i)) if succ(i) exists, else j_i;      out[0] = V(0)
// Every j_i depends only on (key, epoch, i) once the rare Lemire rejections are known
// (RejTable), so the draws are embarrassingly parallel:
//   fy_link  : draw j_i, push i onto target j_i's list (atomicExch linked list)
//   fy_group : per target, sort its (short) writer list -> q[y], succ[] (in place of next)
//   fy_emit  : chase V, write the permutation value straight into the worker stream slot
//              and the inverse permutation inv[e][value] = position (for the histograms).
#include "internal.h"

namespace clairplan {

__global__ void __launch_bounds__(kThreads) fy_link_kernel(uint64_t key, uint32_t F, uint32_t e0,
                                                            uint32_t* __restrict__ head,
                                                            uint32_t* __restrict__ next,
                                                            RejTable rt,
                                                            uint32_t* __restrict__ rej_flag,
                                                            int detect_only, uint32_t i_limit) {
    const uint32_t slot = blockIdx.y;
    const uint32_t e = e0 + slot;
    uint32_t* hd = head + (size_t)slot * F;
    uint32_t* nx = next + (size_t)slot * F;
    const uint32_t er = e - rt.e_base;
    const uint32_t n = rt.count[er];
    const uint32_t* st = rt.step + (size_t)er * rt.cap;
    const uint32_t* cu = rt.cum + (size_t)er * rt.cap;
    const uint32_t lim = i_limit < F ? i_limit : F;
    constexpr int U = 4;  // independent draws + exchanges in flight per thread
    const uint32_t stride = gridDim.x * blockDim.x;
    for (uint32_t i0 = 1 + blockIdx.x * blockDim.x + threadIdx.x; i0 < lim; i0 += U * stride) {
        uint32_t j[U], old[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint32_t i = i0 + u * stride;
            j[u] = kNone;
            if (i < lim) {
                const uint32_t shift = n ? rej_shift(st, cu, n, i) : 0;
                uint32_t extra;
                j[u] = fy_draw(key, e, F, i, shift, &extra);
                if (extra) {
                    bool known = false;
                    for (uint32_t t = 0; t < n; ++t) known |= (st[t] == i);
                    if (!known) atomicMax(&rej_flag[er], i + 1);
                }
            }
        }
        if (detect_only) continue;
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (j[u] != kNone) old[u] = atomicExch(&hd[j[u]], i0 + u * stride);
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (j[u] != kNone) nx[i0 + u * stride] = old[u];
    }
}

// Lists longer than kLocal go through a global scratch area (never seen in practice: the
// expected list length at target y is ~ln(F/y)).
constexpr int kLocal = 48;


// Sorts one target's writer list (>= 3 writers, rare) and links it in place.
__device__ __noinline__ void fy_group_long(uint32_t y, uint32_t a0, uint32_t* nx, uint32_t* qq,
                              uint32_t* scratch, uint32_t scratch_cap, uint32_t* scratch_used,
                              uint32_t* err) {
    uint32_t buf[kLocal];
    uint32_t n = 0;
    uint32_t cur = a0;
    while (cur != kNone && n < (uint32_t)kLocal) {
        int t = (int)n - 1;
        while (t >= 0 && buf[t] > cur) {
            buf[t + 1] = buf[t];
            --t;
        }
        buf[t + 1] = cur;
        ++n;
        cur = nx[cur];
    }
    uint32_t* list = buf;
    if (cur != kNone) {  // overflow: move the whole list to global scratch
        uint32_t m = n;
        for (uint32_t c = cur; c != kNone; c = nx[c]) ++m;
        const uint32_t base = atomicAdd(scratch_used, m);
        if (base + m > scratch_cap) {
            atomicOr(err, 1u);
            return;
        }
        list = scratch + base;
        for (uint32_t t = 0; t < n; ++t) list[t] = buf[t];
        for (uint32_t c = cur; c != kNone; c = nx[c]) {
            int t = (int)n - 1;
            while (t >= 0 && list[t] > c) {
                list[t + 1] = list[t];
                --t;
            }
            list[t + 1] = c;
            ++n;
        }
    }
    qq[y] = (list[0] == y) ? list[1] : list[0];
    for (uint32_t t = 0; t + 1 < n; ++t) nx[list[t]] = list[t + 1];
    nx[list[n - 1]] = kNone;
}

// Per target y: q[y] and the ascending writer chain (succ) in place of the exchange list.
// Each thread walks kGU targets at once (their dependent list loads overlap) and resolves the
// common 0/1/2-writer lists in registers; >= 3 writers go through a register network of up to
// kReg writers, longer lists (small y only) through local memory / global scratch.
constexpr int kGU = 4;
constexpr int kReg = 8;

__device__ __noinline__ void fy_group_mid(uint32_t y, uint32_t a0, uint32_t a1, uint32_t a2,
                                          uint32_t* nx, uint32_t* qq, uint32_t* scratch,
                                          uint32_t scratch_cap, uint32_t* scratch_used,
                                          uint32_t* err) {
    uint32_t a[kReg + 1];
    a[0] = a0;
    a[1] = a1;
    a[2] = a2;
#pragma unroll
    for (int t = 3; t <= kReg; ++t) a[t] = a[t - 1] != kNone ? nx[a[t - 1]] : kNone;
    if (a[kReg] != kNone) {
        fy_group_long(y, a0, nx, qq, scratch, scratch_cap, scratch_used, err);
        return;
    }
    uint32_t qv = kNone;
#pragma unroll
    for (int t = 0; t < kReg; ++t) {
        const uint32_t x = a[t];
        if (x != kNone && x != y && x < qv) qv = x;
    }
    qq[y] = qv;
#pragma unroll
    for (int t = 0; t < kReg; ++t) {
        const uint32_t x = a[t];
        if (x == kNone) continue;
        uint32_t sc = kNone;
#pragma unroll
        for (int r = 0; r < kReg; ++r) {
            const uint32_t z = a[r];
            if (z != kNone && z > x && z < sc) sc = z;
        }
        if (sc != a[t + 1]) nx[x] = sc;
    }
}

__global__ void __launch_bounds__(kThreads) fy_group_kernel(uint32_t F,
                                                             const uint32_t* __restrict__ head,
                                                             uint32_t* __restrict__ next,
                                                             uint32_t* __restrict__ q,
                                                             uint32_t* __restrict__ scratch,
                                                             uint32_t scratch_cap,
                                                             uint32_t* __restrict__ scratch_used,
                                                             uint32_t* __restrict__ err) {
    const uint32_t slot = blockIdx.y;
    const uint32_t* hd = head + (size_t)slot * F;
    uint32_t* nx = next + (size_t)slot * F;
    uint32_t* qq = q + (size_t)slot * F;
    const uint32_t stride = gridDim.x * blockDim.x;
    for (uint32_t y0 = blockIdx.x * blockDim.x + threadIdx.x; y0 < F; y0 += kGU * stride) {
        uint32_t a0[kGU], a1[kGU], a2[kGU];
#pragma unroll
        for (int u = 0; u < kGU; ++u) {
            const uint32_t y = y0 + u * stride;
            a0[u] = y < F ? hd[y] : kNone;
        }
#pragma unroll
        for (int u = 0; u < kGU; ++u) a1[u] = a0[u] != kNone ? nx[a0[u]] : kNone;
#pragma unroll
        for (int u = 0; u < kGU; ++u) a2[u] = a1[u] != kNone ? nx[a1[u]] : kNone;
#pragma unroll
        for (int u = 0; u < kGU; ++u) {
            const uint32_t y = y0 + u * stride;
            if (y >= F) break;
            if (a0[u] == kNone) {
                qq[y] = kNone;
            } else if (a1[u] == kNone) {  // one writer; its succ is already kNone
                qq[y] = (a0[u] == y) ? kNone : a0[u];
            } else if (a2[u] == kNone) {  // two writers: list a0 -> a1, needs ascending order
                const uint32_t lo = min(a0[u], a1[u]), hi = max(a0[u], a1[u]);
                qq[y] = (lo == y) ? hi : lo;
                if (a0[u] > a1[u]) {
                    nx[a1[u]] = a0[u];
                    nx[a0[u]] = kNone;
                }
            } else {
                fy_group_mid(y, a0[u], a1[u], a2[u], nx, qq, scratch, scratch_cap, scratch_used, err);
            }
        }
    }
}

__global__ void __launch_bounds__(kThreads) fy_emit_kernel(uint64_t key, Part part, uint32_t e0,
                                                            const uint32_t* __restrict__ succ,
                                                            const uint32_t* __restrict__ q,
                                                            RejTable rt,
                                                            uint32_t* __restrict__ inv,
                                                            uint32_t* __restrict__ stream,
                                                            uint32_t* __restrict__ perm_out) {
    const uint32_t slot = blockIdx.y;
    const uint32_t e = e0 + slot;
    const uint32_t F = part.F;
    const uint32_t* sc = succ + (size_t)slot * F;
    const uint32_t* qq = q + (size_t)slot * F;
    const uint32_t er = e - rt.e_base;
    const uint32_t n = rt.count[er];
    const uint32_t* st = rt.step + (size_t)er * rt.cap;
    const uint32_t* cu = rt.cum + (size_t)er * rt.cap;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < F; i += gridDim.x * blockDim.x) {
        uint32_t v;
        uint32_t x = kNone;
        if (i == 0) {
            x = 0;
        } else {
            const uint32_t s = sc[i];
            if (s == kNone) {
                uint32_t extra;
                v = fy_draw(key, e, F, i, n ? rej_shift(st, cu, n, i) : 0, &extra);
            } else {
                x = s;
            }
        }
        if (x != kNone) {
            uint32_t nq = qq[x];
            while (nq != kNone) {
                x = nq;
                nq = qq[x];
            }
            v = x;
        }
        if (perm_out) perm_out[(size_t)slot * F + i] = v;
        if (inv) inv[(size_t)e * pitch16(F) + v] = i;
        if (stream && i < part.P) {
            uint32_t w;
            uint64_t spos;
            part.locate(i, e, w, spos);
            if (w >= part.wbegin && w < part.wend) stream[part.stream_offset(w) + spos] = v;
        }
    }
}

// Streams + inverse permutations from externally supplied permutation rows (multi-GPU: rows
// computed on other GPUs and all-gathered over NVLink).  perms[e][p] = value at position p.
__global__ void __launch_bounds__(kThreads) perm_scatter_kernel(Part part, const uint32_t* __restrict__ perms,
                                                                 uint32_t* __restrict__ inv,
                                                                 uint32_t* __restrict__ stream) {
    const uint32_t e = blockIdx.y;
    const uint32_t F = part.F;
    const uint32_t* row = perms + (size_t)e * F;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < F; i += gridDim.x * blockDim.x) {
        const uint32_t v = __ldcs(row + i);
        inv[(size_t)e * pitch16(F) + v] = i;
        if (i < part.P) {
            uint32_t w;
            uint64_t spos;
            part.locate(i, e, w, spos);
            if (w >= part.wbegin && w < part.wend) stream[part.stream_offset(w) + spos] = v;
        }
    }
}

void launch_perm_scatter(cudaStream_t s, const Part& part, const uint32_t* perms, uint32_t* inv,
                         uint32_t* stream) {
    dim3 grid(grid_for(part.F, kThreads * 4, 148u * 16u), part.E);
    perm_scatter_kernel<<<grid, kThreads, 0, s>>>(part, perms, inv, stream);
}

// ---- host launchers ------------------------------------------------------------------
void launch_fy_link(cudaStream_t s, uint64_t key, uint32_t F, uint32_t e0, uint32_t ne,
                    uint32_t* head, uint32_t* next, const RejTable& rt, uint32_t* rej_flag,
                    bool detect_only, uint32_t i_limit) {
    dim3 grid(grid_for(F, kThreads * 4, 148u * 16u), ne);
    fy_link_kernel<<<grid, kThreads, 0, s>>>(key, F, e0, head, next, rt, rej_flag,
                                             detect_only ? 1 : 0, i_limit);
}

void launch_fy_group(cudaStream_t s, uint32_t F, uint32_t ne, const uint32_t* head,
                     uint32_t* next, uint32_t* q, uint32_t* scratch, uint32_t scratch_cap,
                     uint32_t* scratch_used, uint32_t* err) {
    dim3 grid(grid_for(F, kThreads * 4, 148u * 16u), ne);
    fy_group_kernel<<<grid, kThreads, 0, s>>>(F, head, next, q, scratch, scratch_cap,
                                              scratch_used, err);
}

void launch_fy_emit(cudaStream_t s, uint64_t key, const Part& part, uint32_t e0, uint32_t ne,
                    const uint32_t* succ, const uint32_t* q, const RejTable& rt, uint32_t* inv,
                    uint32_t* stream, uint32_t* perm_out) {
    dim3 grid(grid_for(part.F, kThreads * 4, 148u * 16u), ne);
    fy_emit_kernel<<<grid, kThreads, 0, s>>>(key, part, e0, succ, q, rt, inv, stream, perm_out);
}

}  // namespace clairplan
