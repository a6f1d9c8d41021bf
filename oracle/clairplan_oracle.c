/* TEST INFRASTRUCTURE ONLY — see clairplan_oracle.h.
 *
 * Plain-C restatement of the NoPFS clairvoyant plan build of the reference
 * (clairsim, /root/reference/proj).  Every function names the reference lines it
 * follows.  Dense per-worker O(F) tables are used exactly like the reference, one
 * worker at a time, so this is meant for the small/medium parity configurations.
 */
#define _GNU_SOURCE
#include "clairplan_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static __thread char g_err[256];

const char* orc_last_error(void) { return g_err; }

/* rng.hpp:16-25 */
static const uint64_t kGolden = 0x9e3779b97f4a7c15ULL;
uint64_t orc_mix64(uint64_t z) {
    z ^= z >> 30;
    z *= 0xbf58476d1ce4e5b9ULL;
    z ^= z >> 27;
    z *= 0x94d049bb133111ebULL;
    z ^= z >> 31;
    return z;
}

/* rng.hpp:29-34 */
static const uint64_t kPermTag = 0x7065726dULL;
static const uint64_t kSizeTag = 0x73697a65ULL;
uint64_t orc_derive_key(uint64_t seed, uint64_t tag) { return orc_mix64(seed ^ orc_mix64(tag)); }

/* rng.hpp:45-47: position pre-incremented, out = mix64(key + pos * golden) */
static uint64_t next_draw(uint64_t key, uint64_t* pos) {
    *pos += 1;
    return orc_mix64(key + *pos * kGolden);
}

/* rng.hpp:50-63: Lemire multiply-shift with rejection; the 64-bit modulo only when lo < n */
uint64_t orc_bounded(uint64_t key, uint64_t* pos, uint64_t n) {
    uint64_t x = next_draw(key, pos);
    unsigned __int128 m = (unsigned __int128)x * n;
    uint64_t lo = (uint64_t)m;
    if (lo < n) {
        const uint64_t t = (0 - n) % n;
        while (lo < t) {
            x = next_draw(key, pos);
            m = (unsigned __int128)x * n;
            lo = (uint64_t)m;
        }
    }
    return (uint64_t)(m >> 64);
}

/* access.cpp:10,52-57 + rng.cpp:15-24: epoch e starts at stream position e << 34;
 * Fisher-Yates for i = F-1 .. 1 with j = bounded(i + 1). */
int orc_epoch_permutation(uint64_t seed, uint32_t epoch, uint32_t F, uint32_t* a) {
    if (F < 1) {
        snprintf(g_err, sizeof g_err, "permutation needs samples >= 1");
        return 22;
    }
    const uint64_t key = orc_derive_key(seed, kPermTag);
    uint64_t pos = (uint64_t)epoch << 34;
    for (uint32_t i = 0; i < F; ++i) a[i] = i;
    for (uint32_t i = F - 1; i > 0; --i) {
        const uint32_t j = (uint32_t)orc_bounded(key, &pos, (uint64_t)i + 1);
        const uint32_t t = a[i];
        a[i] = a[j];
        a[j] = t;
    }
    return 0;
}

/* Same shuffle with the Lemire rejection loop removed (test-only counterfactual: shows that a
 * rejection KAT really exercises rng.hpp:54-60). */
int orc_epoch_permutation_norej(uint64_t seed, uint32_t epoch, uint32_t F, uint32_t* a) {
    const uint64_t key = orc_derive_key(seed, kPermTag);
    uint64_t pos = (uint64_t)epoch << 34;
    for (uint32_t i = 0; i < F; ++i) a[i] = i;
    for (uint32_t i = F - 1; i > 0; --i) {
        const uint64_t x = next_draw(key, &pos);
        const uint32_t j = (uint32_t)(((unsigned __int128)x * ((uint64_t)i + 1)) >> 64);
        const uint32_t t = a[i];
        a[i] = a[j];
        a[j] = t;
    }
    return 0;
}

/* access.cpp:33-39 */
void orc_batch_slice(uint64_t batch_size, uint32_t workers, uint32_t worker, uint64_t* begin,
                     uint64_t* end) {
    const uint64_t base = batch_size / workers;
    const uint64_t extra = batch_size % workers;
    const uint64_t b = (uint64_t)worker * base + (worker < extra ? worker : extra);
    *begin = b;
    *end = b + base + (worker < extra ? 1 : 0);
}

/* rng.cpp:7-13 (CounterRng::normal, cosine branch) */
static double normal_draw(uint64_t key, uint64_t* pos) {
    const double u1 = (double)(next_draw(key, pos) >> 11) * 0x1.0p-53;
    const double u2 = (double)(next_draw(key, pos) >> 11) * 0x1.0p-53;
    const double r = sqrt(-2.0 * log(1.0 - u1));
    return r * cos(2.0 * M_PI * u2);
}

/* perfmodel.cpp:68-99 (DatasetModel::generate) — host-side input generation */
int orc_generate_sizes(uint64_t F, double mean, double sigma_in, int has_total, double total,
                       uint64_t seed, int sigma_relative, double* s) {
    if (F < 1 || mean <= 0 || sigma_in < 0) {
        snprintf(g_err, sizeof g_err, "invalid dataset parameters");
        return 22;
    }
    const double sigma = sigma_relative ? sigma_in * mean : sigma_in;
    double floor_mb = mean / 100.0;
    if (floor_mb < 1e-3) floor_mb = 1e-3;
    if (floor_mb > mean) floor_mb = mean;
    const uint64_t key = orc_derive_key(seed, kSizeTag);
    uint64_t pos = 0;
    double sum = 0;
    for (uint64_t k = 0; k < F; ++k) {
        double v;
        if (sigma == 0) {
            v = mean;
        } else {
            const double x = mean + sigma * normal_draw(key, &pos);
            v = (floor_mb < x) ? x : floor_mb; /* std::max(floor, x) = (floor < x) ? x : floor */
        }
        s[k] = v;
        sum += v;
    }
    if (has_total) {
        const double scale = total / sum;
        for (uint64_t k = 0; k < F; ++k) s[k] *= scale;
    }
    return 0;
}

struct orc_plan {
    uint32_t N, F, J;
    uint32_t* entries;       /* worker-major streams */
    uint64_t* stream_off;    /* [N+1] */
    uint32_t* class_entries; /* (w, j) major class lists */
    uint64_t* class_off;     /* [N*J+1] */
    uint64_t* holder_off;    /* [F+1] */
    uint32_t* holders;       /* 3 x u32 per holder */
};

/* access.cpp:41-50 (PartitionSpec::validate), messages verbatim */
static int validate(uint64_t F, uint32_t N, uint32_t B, uint32_t E) {
    if (F < 1) return snprintf(g_err, sizeof g_err, "dataset must have at least one sample"), 22;
    if (N < 1) return snprintf(g_err, sizeof g_err, "num_workers must be >= 1"), 22;
    if (E < 1) return snprintf(g_err, sizeof g_err, "epochs must be >= 1"), 22;
    if (B < N) return snprintf(g_err, sizeof g_err, "global batch must be >= num_workers"), 22;
    if (B > F)
        return snprintf(g_err, sizeof g_err, "global batch %u exceeds dataset size %llu", B,
                        (unsigned long long)F),
               22;
    return 0;
}

/* sort keys for policies.cpp:154-160 and :31-36 */
typedef struct {
    uint32_t k, count;
    uint64_t first;
} cand_t;

static int by_count_then_first(const void* a, const void* b) {
    const cand_t* x = a;
    const cand_t* y = b;
    if (x->count != y->count) return x->count > y->count ? -1 : 1;
    if (x->first != y->first) return x->first < y->first ? -1 : 1;
    return x->k < y->k ? -1 : (x->k > y->k); /* stable_sort keeps k order on full ties */
}

static int by_first_then_k(const void* a, const void* b) {
    const cand_t* x = a;
    const cand_t* y = b;
    if (x->first != y->first) return x->first < y->first ? -1 : 1;
    return x->k < y->k ? -1 : (x->k > y->k);
}

/* policies.cpp:144-166 (nopfs_assign_caches) + :16-23 (first_access_positions) + :40-55
 * (pack_first_fit, sequential double remaining[j] -= s) + :31-36 (order_by_first_access)
 * + :124-142 (build_index, here with u64 offsets). counts_of(w) gives dense counts. */
static int assign(orc_plan* p, const double* caps, const double* sizes,
                  const uint32_t* dense_counts /* may be NULL: recount from streams */) {
    const uint32_t N = p->N, F = p->F, J = p->J;
    const uint64_t NOIDX = UINT64_MAX;
    uint32_t* counts = malloc(sizeof(uint32_t) * (size_t)F);
    uint64_t* first = malloc(sizeof(uint64_t) * (size_t)F);
    cand_t* cand = malloc(sizeof(cand_t) * (size_t)F);
    uint32_t* cls = malloc(sizeof(uint32_t) * (size_t)F);
    size_t cap_entries = 1024, used = 0;
    p->class_entries = malloc(sizeof(uint32_t) * cap_entries);
    p->class_off = calloc((size_t)N * J + 1, sizeof(uint64_t));
    double* remaining = malloc(sizeof(double) * (J ? J : 1));
    for (uint32_t w = 0; w < N && J > 0; ++w) {
        const uint32_t* st = p->entries + p->stream_off[w];
        const uint64_t L = p->stream_off[w + 1] - p->stream_off[w];
        if (dense_counts) {
            memcpy(counts, dense_counts + (uint64_t)w * F, sizeof(uint32_t) * F);
        } else { /* access.cpp:80-88 over all epochs */
            memset(counts, 0, sizeof(uint32_t) * F);
            for (uint64_t i = 0; i < L; ++i) counts[st[i]]++;
        }
        for (uint32_t k = 0; k < F; ++k) first[k] = NOIDX;
        for (uint64_t i = 0; i < L; ++i)
            if (first[st[i]] == NOIDX) first[st[i]] = i;
        size_t n = 0;
        for (uint32_t k = 0; k < F; ++k)
            if (counts[k] > 0) cand[n++] = (cand_t){k, counts[k], first[k]};
        qsort(cand, n, sizeof(cand_t), by_count_then_first);
        for (uint32_t j = 0; j < J; ++j) remaining[j] = caps[j];
        for (size_t c = 0; c < n; ++c) {
            const double s = sizes[cand[c].k];
            cls[c] = 0;
            for (uint32_t j = 0; j < J; ++j) {
                if (s <= remaining[j]) {
                    remaining[j] -= s;
                    cls[c] = j + 1;
                    break;
                }
            }
        }
        for (uint32_t j = 0; j < J; ++j) {
            size_t m = 0;
            for (size_t c = 0; c < n; ++c)
                if (cls[c] == j + 1) ++m;
            cand_t* list = malloc(sizeof(cand_t) * (m ? m : 1));
            m = 0;
            for (size_t c = 0; c < n; ++c)
                if (cls[c] == j + 1) list[m++] = cand[c];
            qsort(list, m, sizeof(cand_t), by_first_then_k);
            if (used + m > cap_entries) {
                while (used + m > cap_entries) cap_entries *= 2;
                p->class_entries = realloc(p->class_entries, sizeof(uint32_t) * cap_entries);
            }
            for (size_t i = 0; i < m; ++i) p->class_entries[used + i] = list[i].k;
            used += m;
            p->class_off[(uint64_t)w * J + j + 1] = used;
            free(list);
        }
    }
    for (uint64_t i = 1; i <= (uint64_t)N * J; ++i)
        if (p->class_off[i] < p->class_off[i - 1]) p->class_off[i] = p->class_off[i - 1];
    /* build_index, policies.cpp:124-142 */
    p->holder_off = calloc((size_t)F + 1, sizeof(uint64_t));
    for (uint64_t i = 0; i < used; ++i) p->holder_off[p->class_entries[i] + 1]++;
    for (uint32_t k = 0; k < F; ++k) p->holder_off[k + 1] += p->holder_off[k];
    p->holders = malloc(sizeof(uint32_t) * 3 * (used ? used : 1));
    uint64_t* cursor = malloc(sizeof(uint64_t) * ((size_t)F + 1));
    memcpy(cursor, p->holder_off, sizeof(uint64_t) * ((size_t)F + 1));
    for (uint32_t w = 0; w < N; ++w)
        for (uint32_t j = 0; j < J; ++j) {
            const uint64_t b = p->class_off[(uint64_t)w * J + j];
            const uint64_t e = p->class_off[(uint64_t)w * J + j + 1];
            for (uint64_t i = b; i < e; ++i) {
                const uint64_t slot = cursor[p->class_entries[i]]++;
                p->holders[3 * slot + 0] = w;
                p->holders[3 * slot + 1] = j + 1;
                p->holders[3 * slot + 2] = (uint32_t)(i - b);
            }
        }
    free(cursor);
    free(remaining);
    free(cls);
    free(cand);
    free(first);
    free(counts);
    return 0;
}

/* access.cpp:59-78 (build_access_streams, for_each_worker_slice :14-29) */
orc_plan* orc_plan_build(uint64_t seed, uint32_t F, uint32_t N, uint32_t B, uint32_t E,
                         int drop_last, uint32_t J, const double* caps, const double* sizes) {
    if (validate(F, N, B, E)) return NULL;
    orc_plan* p = calloc(1, sizeof(orc_plan));
    p->N = N;
    p->F = F;
    p->J = J;
    const uint64_t full = F / B;
    const uint64_t tail = drop_last ? 0 : F % B;
    const uint64_t nb = full + (tail > 0);
    uint64_t* len = calloc(N, sizeof(uint64_t));
    for (uint64_t h = 0; h < nb; ++h)
        for (uint32_t w = 0; w < N; ++w) {
            uint64_t b, e;
            orc_batch_slice(h < full ? B : tail, N, w, &b, &e);
            len[w] += (e - b) * E;
        }
    p->stream_off = calloc((size_t)N + 1, sizeof(uint64_t));
    for (uint32_t w = 0; w < N; ++w) p->stream_off[w + 1] = p->stream_off[w] + len[w];
    p->entries = malloc(sizeof(uint32_t) * (p->stream_off[N] ? p->stream_off[N] : 1));
    uint32_t* perm = malloc(sizeof(uint32_t) * F);
    uint64_t* cur = malloc(sizeof(uint64_t) * N);
    memcpy(cur, p->stream_off, sizeof(uint64_t) * N);
    for (uint32_t ep = 0; ep < E; ++ep) {
        orc_epoch_permutation(seed, ep, F, perm);
        for (uint64_t h = 0; h < nb; ++h)
            for (uint32_t w = 0; w < N; ++w) {
                uint64_t b, e;
                orc_batch_slice(h < full ? B : tail, N, w, &b, &e);
                memcpy(p->entries + cur[w], perm + h * B + b, sizeof(uint32_t) * (e - b));
                cur[w] += e - b;
            }
    }
    free(cur);
    free(perm);
    free(len);
    assign(p, caps, sizes, NULL);
    return p;
}

orc_plan* orc_assign_from_streams(uint32_t N, uint32_t F, const uint32_t* entries,
                                  const uint64_t* offsets, const uint32_t* counts, uint32_t J,
                                  const double* caps, const double* sizes) {
    orc_plan* p = calloc(1, sizeof(orc_plan));
    p->N = N;
    p->F = F;
    p->J = J;
    p->stream_off = malloc(sizeof(uint64_t) * ((size_t)N + 1));
    memcpy(p->stream_off, offsets, sizeof(uint64_t) * ((size_t)N + 1));
    p->entries = malloc(sizeof(uint32_t) * (offsets[N] ? offsets[N] : 1));
    memcpy(p->entries, entries, sizeof(uint32_t) * offsets[N]);
    assign(p, caps, sizes, counts);
    return p;
}

uint64_t orc_plan_stream(const orc_plan* p, uint32_t w, const uint32_t** data) {
    *data = p->entries + p->stream_off[w];
    return p->stream_off[w + 1] - p->stream_off[w];
}

uint64_t orc_plan_class_list(const orc_plan* p, uint32_t w, uint32_t j, const uint32_t** data) {
    const uint64_t i = (uint64_t)w * p->J + j;
    *data = p->class_entries + p->class_off[i];
    return p->class_off[i + 1] - p->class_off[i];
}

uint64_t orc_plan_holders(const orc_plan* p, const uint64_t** offsets, const uint32_t** holders) {
    *offsets = p->holder_off;
    *holders = p->holders;
    return p->holder_off[p->F];
}

void orc_plan_free(orc_plan* p) {
    if (!p) return;
    free(p->entries);
    free(p->stream_off);
    free(p->class_entries);
    free(p->class_off);
    free(p->holder_off);
    free(p->holders);
    free(p);
}
