// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// C-ABI harness around the UNMODIFIED reference sources (clairsim, compiled from
// /root/reference/proj/src by oracle/Makefile into oracle/_ref/). Only tests/,
// __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg may
// load the resulting library; it is the checker and the CPU baseline, never the
// thing measured as the product.
//
// Two ways to run the reference plan:
//   mode 0 "verbatim":   build_access_streams -> access_frequencies (every worker) ->
//                        nopfs_assign_caches, exactly policies.cpp:446-456.
//   mode 1 "per-worker": the reference's own epoch_permutation / batch_slice /
//                        access_frequencies / nopfs_assign_caches called one worker at a
//                        time on all host threads, then the reference's own
//                        CacheAssignment::build_index over the merged class lists.
//                        Streams are cut like for_each_worker_slice (access.cpp:14-29,
//                        anonymous namespace, so restated here).  tests/ check mode 1 ==
//                        mode 0 before it is trusted for large configs / the baseline.
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <optional>
#include <string>
#include <thread>
#include <vector>

#include "clairsim/access.hpp"
#include "clairsim/analysis.hpp"
#include "clairsim/perfmodel.hpp"
#include "clairsim/policies.hpp"
#include "clairsim/rng.hpp"
#include "clairsim/scenarios.hpp"

using namespace clairsim;

namespace {

thread_local std::string g_err;
// wall-clock phases of the last ref_plan_build_subset on this thread (ms): permutations,
// stream cutting, per-worker assignment, build_index (the CPU-baseline sample extrapolates
// the assignment phase of a worker subset to all workers)
thread_local double g_phase_ms[4] = {0, 0, 0, 0};

double now_ms() {
    return std::chrono::duration<double, std::milli>(
               std::chrono::steady_clock::now().time_since_epoch()).count();
}

struct RefPlan {
    uint32_t F = 0;
    std::vector<AccessStream> streams;
    CacheAssignment assign;
    std::vector<FrequencyTable> freqs;  // verbatim mode only (dense N x F)
    std::vector<uint32_t> holders_flat;  // 3 x u32 per holder, AoS like Holder
};

SystemConfig make_cfg(uint32_t workers, uint32_t J, const double* caps) {
    // Only cfg.workers and storage[1..J].capacity_mb are read by nopfs_assign_caches
    // (policies.cpp:144-166); staging (class 0) capacity is never packed.
    SystemConfig cfg;
    cfg.workers = workers;
    StorageClassSpec staging;
    staging.name = "staging";
    staging.capacity_mb = 1;
    cfg.storage.push_back(staging);
    for (uint32_t j = 0; j < J; ++j) {
        StorageClassSpec sc;
        sc.name = "class" + std::to_string(j + 1);
        sc.capacity_mb = caps[j];
        cfg.storage.push_back(sc);
    }
    return cfg;
}

template <typename Fn>
void parallel_for(uint64_t n, int threads, Fn&& fn) {
    if (threads <= 1 || n <= 1) {
        for (uint64_t i = 0; i < n; ++i) fn(i);
        return;
    }
    std::atomic<uint64_t> next{0};
    std::vector<std::thread> pool;
    for (int t = 0; t < threads; ++t)
        pool.emplace_back([&] {
            for (uint64_t i = next++; i < n; i = next++) fn(i);
        });
    for (auto& th : pool) th.join();
}

void flatten_holders(RefPlan& p) {
    p.holders_flat.resize(p.assign.holders.size() * 3);
    for (size_t i = 0; i < p.assign.holders.size(); ++i) {
        p.holders_flat[3 * i + 0] = p.assign.holders[i].worker;
        p.holders_flat[3 * i + 1] = p.assign.holders[i].storage_class;
        p.holders_flat[3 * i + 2] = p.assign.holders[i].position;
    }
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

void ref_last_phase_ms(double* out) {
    for (int i = 0; i < 4; ++i) out[i] = g_phase_ms[i];
}

// CounterRng stream values (rng.hpp:36-47).
int ref_rng_stream(uint64_t seed, uint64_t tag, uint64_t start, uint64_t n, uint64_t* out) {
    CounterRng rng = CounterRng::for_stream(seed, tag, start);
    for (uint64_t i = 0; i < n; ++i) out[i] = rng.next();
    return 0;
}

// CounterRng::bounded (rng.hpp:50-63): draws n values, also reports stream positions.
int ref_rng_bounded(uint64_t key, uint64_t start, uint64_t bound, uint64_t n, uint64_t* out,
                    uint64_t* pos_after) {
    CounterRng rng(key, start);
    for (uint64_t i = 0; i < n; ++i) out[i] = rng.bounded(bound);
    if (pos_after) *pos_after = rng.position();
    return 0;
}

int ref_epoch_permutation(uint64_t seed, uint32_t epoch, uint32_t F, uint32_t* out) {
    try {
        const auto p = epoch_permutation(Seed{seed}, epoch, F);
        std::memcpy(out, p.data(), p.size() * sizeof(uint32_t));
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 22;
    }
}

// batch_slice (access.cpp:33-39).
void ref_batch_slice(uint64_t batch_size, uint32_t workers, uint32_t worker, uint64_t* begin,
                     uint64_t* end) {
    const auto [b, e] = batch_slice(batch_size, workers, worker);
    *begin = b;
    *end = e;
}

int ref_partition_validate(uint64_t samples, uint32_t N, uint32_t B, uint32_t E, int drop_last) {
    try {
        PartitionSpec part{N, B, E, drop_last != 0};
        part.validate(samples);
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 22;
    }
}

// DatasetModel::generate (perfmodel.cpp:68-99) -> sizes.
int ref_generate_sizes(uint64_t F, double mean, double sigma, int has_total, double total,
                       uint64_t seed, int sigma_relative, double* out, double* total_out) {
    try {
        std::optional<double> t;
        if (has_total) t = total;
        const auto d = DatasetModel::generate(F, mean, sigma, t, seed, sigma_relative != 0);
        std::memcpy(out, d.sizes_mb.data(), F * sizeof(double));
        if (total_out) *total_out = d.total_mb;
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 22;
    }
}

// Full reference plan. mode 0 = verbatim, mode 1 = per-worker decomposition on `threads`.
void* ref_plan_build_subset(uint64_t seed, uint32_t F, uint32_t N, uint32_t B, uint32_t E,
                            int drop_last, uint32_t J, const double* caps, const double* sizes,
                            int threads, const uint32_t* subset, uint32_t nsubset);

void* ref_plan_build(uint64_t seed, uint32_t F, uint32_t N, uint32_t B, uint32_t E,
                     int drop_last, uint32_t J, const double* caps, const double* sizes,
                     int mode, int threads) {
    if (mode == 1) return ref_plan_build_subset(seed, F, N, B, E, drop_last, J, caps, sizes,
                                                threads, nullptr, 0);
    try {
        auto p = std::make_unique<RefPlan>();
        p->F = F;
        PartitionSpec part{N, B, E, drop_last != 0};
        const DatasetModel dataset = DatasetModel::from_sizes(std::vector<double>(sizes, sizes + F));
        if (mode == 0) {
            const SystemConfig cfg = make_cfg(N, J, caps);
            p->streams = build_access_streams(Seed{seed}, F, part);
            p->freqs.reserve(N);
            for (const auto& st : p->streams)
                p->freqs.push_back(access_frequencies(st, F, 0, st.epoch_count()));
            p->assign = nopfs_assign_caches(p->freqs, cfg, dataset, p->streams);
        }
        flatten_holders(*p);
        return p.release();
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}

// Per-worker decomposition restricted to a worker subset (the others' class lists stay empty,
// so build_index yields the holder CSR restricted to the subset: a subsequence of the full
// CSR because holders are worker-ordered).  subset == nullptr: all workers.
void* ref_plan_build_subset(uint64_t seed, uint32_t F, uint32_t N, uint32_t B, uint32_t E,
                            int drop_last, uint32_t J, const double* caps, const double* sizes,
                            int threads, const uint32_t* subset, uint32_t nsubset) {
    try {
        auto p = std::make_unique<RefPlan>();
        p->F = F;
        PartitionSpec part{N, B, E, drop_last != 0};
        const DatasetModel dataset = DatasetModel::from_sizes(std::vector<double>(sizes, sizes + F));
        part.validate(F);
        double t0 = now_ms();
        std::vector<std::vector<uint32_t>> perms(E);
        parallel_for(E, threads, [&](uint64_t e) {
            perms[e] = epoch_permutation(Seed{seed}, static_cast<uint32_t>(e), F);
        });
        double t1 = now_ms();
        g_phase_ms[0] = t1 - t0;
        const uint64_t full = F / B;
        const uint64_t tail = part.drop_last ? 0 : F % B;
        const uint64_t nb = full + (tail > 0 ? 1 : 0);
        p->streams.resize(N);
        parallel_for(N, threads, [&](uint64_t w) {
            auto& st = p->streams[w];
            st.worker_id = static_cast<uint32_t>(w);
            st.epoch_offsets.push_back(0);
            st.batch_offsets.push_back(0);
            for (uint32_t e = 0; e < E; ++e) {
                for (uint64_t h = 0; h < nb; ++h) {
                    const uint64_t bs = h < full ? B : tail;
                    const auto [sb, se] = batch_slice(bs, N, static_cast<uint32_t>(w));
                    st.entries.insert(st.entries.end(), perms[e].begin() + h * B + sb,
                                      perms[e].begin() + h * B + se);
                    st.batch_offsets.push_back(st.entries.size());
                }
                st.epoch_offsets.push_back(st.entries.size());
            }
        });
        t0 = now_ms();
        g_phase_ms[1] = t0 - t1;
        perms.clear();
        perms.shrink_to_fit();
        p->assign.class_lists.assign(N, std::vector<std::vector<uint32_t>>(J));
        const SystemConfig cfg1 = make_cfg(1, J, caps);
        std::vector<uint32_t> todo;
        if (subset) todo.assign(subset, subset + nsubset);
        else for (uint32_t w = 0; w < N; ++w) todo.push_back(w);
        parallel_for(todo.size(), threads, [&](uint64_t i) {
            const uint32_t w = todo[i];
            const auto& st = p->streams[w];
            const auto freq = access_frequencies(st, F, 0, st.epoch_count());
            auto one = nopfs_assign_caches({freq}, cfg1, dataset, {st});
            if (J > 0) p->assign.class_lists[w] = std::move(one.class_lists[0]);
        });
        t1 = now_ms();
        g_phase_ms[2] = t1 - t0;
        p->assign.build_index(F);
        g_phase_ms[3] = now_ms() - t1;
        flatten_holders(*p);
        return p.release();
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}

// Worker-subset plan for datasets whose permutations do not fit host memory together
// (config 5: 100 x 100 M samples): epochs are generated one per thread at a time and only the
// subset workers' slices are kept; the other workers' streams stay empty.
void* ref_plan_build_subset_lowmem(uint64_t seed, uint32_t F, uint32_t N, uint32_t B, uint32_t E,
                                   int drop_last, uint32_t J, const double* caps,
                                   const double* sizes, int threads, const uint32_t* subset,
                                   uint32_t nsubset) {
    try {
        auto p = std::make_unique<RefPlan>();
        p->F = F;
        PartitionSpec part{N, B, E, drop_last != 0};
        const DatasetModel dataset = DatasetModel::from_sizes(std::vector<double>(sizes, sizes + F));
        part.validate(F);
        const uint64_t full = F / B;
        const uint64_t tail = part.drop_last ? 0 : F % B;
        const uint64_t nb = full + (tail > 0 ? 1 : 0);
        // per (subset worker, epoch) slices, the same insert order as build_access_streams
        std::vector<std::vector<std::vector<uint32_t>>> part_e(nsubset,
                                                               std::vector<std::vector<uint32_t>>(E));
        parallel_for(E, threads, [&](uint64_t e) {
            const auto perm = epoch_permutation(Seed{seed}, static_cast<uint32_t>(e), F);
            for (uint32_t i = 0; i < nsubset; ++i) {
                auto& out = part_e[i][e];
                for (uint64_t h = 0; h < nb; ++h) {
                    const uint64_t bs = h < full ? B : tail;
                    const auto [sb, se] = batch_slice(bs, N, subset[i]);
                    out.insert(out.end(), perm.begin() + h * B + sb, perm.begin() + h * B + se);
                }
            }
        });
        p->streams.resize(N);
        for (uint32_t w = 0; w < N; ++w) {
            p->streams[w].worker_id = w;
            p->streams[w].epoch_offsets.push_back(0);
            p->streams[w].batch_offsets.push_back(0);
        }
        for (uint32_t i = 0; i < nsubset; ++i) {
            auto& st = p->streams[subset[i]];
            st.epoch_offsets.clear();
            st.epoch_offsets.push_back(0);
            for (uint32_t e = 0; e < E; ++e) {
                st.entries.insert(st.entries.end(), part_e[i][e].begin(), part_e[i][e].end());
                st.epoch_offsets.push_back(st.entries.size());
                std::vector<uint32_t>().swap(part_e[i][e]);
            }
        }
        p->assign.class_lists.assign(N, std::vector<std::vector<uint32_t>>(J));
        const SystemConfig cfg1 = make_cfg(1, J, caps);
        parallel_for(nsubset, threads, [&](uint64_t i) {
            const uint32_t w = subset[i];
            const auto& st = p->streams[w];
            const auto freq = access_frequencies(st, F, 0, st.epoch_count());
            auto one = nopfs_assign_caches({freq}, cfg1, dataset, {st});
            if (J > 0) p->assign.class_lists[w] = std::move(one.class_lists[0]);
        });
        p->assign.build_index(F);
        flatten_holders(*p);
        return p.release();
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}

// nopfs_assign_caches on caller-provided streams + dense frequency tables (policies.hpp:88-90).
// streams: concatenated entries with per-worker offsets [N+1]; counts: N x F dense.
void* ref_assign_from_streams(uint32_t N, uint32_t F, const uint32_t* entries,
                              const uint64_t* offsets, const uint32_t* counts, uint32_t J,
                              const double* caps, const double* sizes) {
    try {
        auto p = std::make_unique<RefPlan>();
        p->F = F;
        const DatasetModel dataset = DatasetModel::from_sizes(std::vector<double>(sizes, sizes + F));
        const SystemConfig cfg = make_cfg(N, J, caps);
        p->streams.resize(N);
        p->freqs.resize(N);
        for (uint32_t w = 0; w < N; ++w) {
            p->streams[w].worker_id = w;
            p->streams[w].entries.assign(entries + offsets[w], entries + offsets[w + 1]);
            p->streams[w].epoch_offsets = {0, p->streams[w].entries.size()};
            p->streams[w].batch_offsets = {0, p->streams[w].entries.size()};
            p->freqs[w].worker_id = w;
            p->freqs[w].counts.assign(counts + static_cast<uint64_t>(w) * F,
                                      counts + static_cast<uint64_t>(w + 1) * F);
        }
        p->assign = nopfs_assign_caches(p->freqs, cfg, dataset, p->streams);
        flatten_holders(*p);
        return p.release();
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}

uint64_t ref_plan_stream(void* h, uint32_t w, const uint32_t** data) {
    auto* p = static_cast<RefPlan*>(h);
    *data = p->streams[w].entries.data();
    return p->streams[w].entries.size();
}

uint64_t ref_plan_epoch_offsets(void* h, uint32_t w, const uint64_t** data) {
    auto* p = static_cast<RefPlan*>(h);
    *data = p->streams[w].epoch_offsets.data();
    return p->streams[w].epoch_offsets.size();
}

uint64_t ref_plan_batch_offsets(void* h, uint32_t w, const uint64_t** data) {
    auto* p = static_cast<RefPlan*>(h);
    *data = p->streams[w].batch_offsets.data();
    return p->streams[w].batch_offsets.size();
}

uint64_t ref_plan_class_list(void* h, uint32_t w, uint32_t j, const uint32_t** data) {
    auto* p = static_cast<RefPlan*>(h);
    const auto& l = p->assign.class_lists[w][j];
    *data = l.data();
    return l.size();
}

// holder_offsets (u32[F+1], policies.hpp:59) and holders flattened {worker, class, position}.
uint64_t ref_plan_holders(void* h, const uint32_t** offsets, const uint32_t** holders) {
    auto* p = static_cast<RefPlan*>(h);
    *offsets = p->assign.holder_offsets.data();
    *holders = p->holders_flat.data();
    return p->assign.holders.size();
}

// access_frequencies (access.cpp:80-88) of worker w over epochs [eb, ee).
int ref_access_frequencies(void* h, uint32_t w, uint32_t eb, uint32_t ee, uint32_t* out) {
    auto* p = static_cast<RefPlan*>(h);
    const auto f = access_frequencies(p->streams[w], p->F, eb, ee);
    std::memcpy(out, f.counts.data(), f.counts.size() * sizeof(uint32_t));
    return 0;
}

int ref_worker_access_counts(uint64_t seed, uint32_t F, uint32_t N, uint32_t B, uint32_t E,
                             int drop_last, uint32_t w, uint32_t* out) {
    try {
        const auto c = worker_access_counts(Seed{seed}, F, PartitionSpec{N, B, E, drop_last != 0}, w);
        std::memcpy(out, c.data(), c.size() * sizeof(uint32_t));
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 22;
    }
}

int ref_all_access_counts(uint64_t seed, uint32_t F, uint32_t N, uint32_t B, uint32_t E,
                          int drop_last, uint32_t* out) {
    try {
        const auto c = all_access_counts(Seed{seed}, F, PartitionSpec{N, B, E, drop_last != 0});
        for (uint32_t w = 0; w < N; ++w)
            std::memcpy(out + static_cast<uint64_t>(w) * F, c[w].data(), F * sizeof(uint32_t));
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 22;
    }
}

// The presets' reference system (scenarios.cpp:15-46, reached through make_scenario: the
// builder is file-local) for N workers with cache classes 1..J of the given capacities
// (class specs beyond the preset's two repeat the last one).
static SystemConfig chooser_cfg(uint32_t N, uint32_t J, const double* caps) {
    SystemConfig cfg = make_scenario("imagenet1k").system;
    cfg.workers = N;
    const StorageClassSpec last = cfg.storage.back();
    cfg.storage.resize(1 + J, last);
    for (uint32_t j = 0; j < J; ++j) cfg.storage[1 + j].capacity_mb = caps[j];
    return cfg;
}

// fetch_time_local / fetch_time_remote (1.0, cfg, j) and fetch_time_pfs (1.0, cfg, gamma):
// the unit times the device chooser compares (perfmodel.cpp:109-121)
int ref_unit_times(uint32_t N, uint32_t J, const double* caps, uint32_t gamma, double* local_t,
                   double* remote_t, double* pfs_t) {
    try {
        const SystemConfig cfg = chooser_cfg(N, J, caps);
        for (uint32_t j = 0; j < J; ++j) {
            local_t[j] = fetch_time_local(1.0, cfg, j + 1);
            remote_t[j] = fetch_time_remote(1.0, cfg, j + 1);
        }
        *pfs_t = fetch_time_pfs(1.0, cfg, gamma);
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 22;
    }
}

// The reference's choose_source (policies.cpp:218-227) per query on the plan's assignment;
// out[3i..3i+2] = {kind (FetchSource::Kind), storage_class, worker}.
int ref_choose_sources(void* h, uint32_t N, uint32_t J, const double* caps, const uint64_t* progress,
                       uint32_t gamma, int allow_local, int allow_remote, int heuristic,
                       uint64_t n, const uint32_t* samples, const uint32_t* workers,
                       uint32_t* out) {
    try {
        auto* p = static_cast<RefPlan*>(h);
        const SystemConfig cfg = chooser_cfg(N, J, caps);
        PrefetchProgress pr;
        pr.completed.assign(N, std::vector<uint64_t>(J, 0));
        for (uint32_t w = 0; w < N; ++w)
            for (uint32_t j = 0; j < J; ++j) pr.completed[w][j] = progress[(uint64_t)w * J + j];
        for (uint64_t i = 0; i < n; ++i) {
            const FetchSource s = choose_source(samples[i], workers[i], p->assign, pr, gamma, cfg,
                                                allow_local != 0, allow_remote != 0, heuristic != 0);
            out[3 * i] = static_cast<uint32_t>(s.kind);
            out[3 * i + 1] = s.storage_class;
            out[3 * i + 2] = s.worker;
        }
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 22;
    }
}

// analysis.cpp:84-96 and the C1 / C2 acceptance quantities (acceptance.cpp:76-158)
int ref_monte_carlo_histogram(uint64_t seed, uint32_t N, uint32_t E, uint32_t F, uint64_t* out) {
    try {
        const FrequencyHistogram h = monte_carlo_histogram(Seed{seed}, N, E, F);
        for (size_t c = 0; c < h.buckets.size(); ++c) out[c] = h.buckets[c];
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 22;
    }
}

double ref_expected_hot_samples(uint32_t N, uint32_t E, uint64_t F, double delta) {
    return expected_hot_samples(AccessDistributionParams{N, E, F, delta});
}

uint32_t ref_hot_count_threshold(uint32_t N, uint32_t E, double delta) {
    return hot_count_threshold(N, E, delta);
}

// {high_threshold, counterpart_low_bound, low_threshold, counterpart_high_bound}
int ref_lemma1_bounds(uint32_t N, uint32_t E, double delta, int64_t* out) {
    try {
        const Lemma1Bounds b = lemma1_bounds(N, E, delta);
        out[0] = b.high_threshold;
        out[1] = b.counterpart_low_bound;
        out[2] = b.low_threshold;
        out[3] = b.counterpart_high_bound;
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 22;
    }
}

void ref_plan_free(void* h) { delete static_cast<RefPlan*>(h); }

}  // extern "C"
