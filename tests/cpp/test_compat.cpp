// Reference test cases for the hot path (proj/tests/test_access.cpp, test_policies.cpp),
// restated and run against libclairsim_b200.so — i.e. against the GPU implementation through
// the reference's own C++ API.  Exit code 0 = all checks passed.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <fstream>
#include <iterator>
#include <numeric>
#include <set>
#include <stdexcept>
#include <string>
#include <vector>

#include "clairsim/access.hpp"
#include "clairsim/policies.hpp"

using namespace clairsim;

static int g_fail = 0, g_checks = 0;
#define CHECK(c)                                                              \
    do {                                                                      \
        ++g_checks;                                                           \
        if (!(c)) {                                                           \
            ++g_fail;                                                         \
            std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #c); \
        }                                                                     \
    } while (0)
#define CHECK_THROWS(expr)                      \
    do {                                        \
        bool thrown_ = false;                   \
        try {                                   \
            expr;                               \
        } catch (const std::invalid_argument&) { \
            thrown_ = true;                     \
        }                                       \
        CHECK(thrown_);                         \
    } while (0)

static std::vector<uint32_t> golden(const std::string& name) {
    std::ifstream in(std::string(GOLDEN_DIR) + "/" + name);
    return {std::istream_iterator<uint32_t>(in), std::istream_iterator<uint32_t>()};
}

static SystemConfig small_system(uint32_t workers, double cap1, double cap2) {
    SystemConfig cfg;  // only workers and storage[1..J].capacity_mb matter to the NoPFS plan
    cfg.workers = workers;
    StorageClassSpec st{"staging", 1000, {}, {}, 1}, ram{"ram", cap1, {}, {}, 1},
        ssd{"ssd", cap2, {}, {}, 1};
    cfg.storage = {st, ram, ssd};
    return cfg;
}

static std::vector<uint64_t> first_pos(const AccessStream& st, uint32_t F) {
    std::vector<uint64_t> f(F, UINT64_MAX);
    for (uint64_t i = 0; i < st.entries.size(); ++i)
        if (f[st.entries[i]] == UINT64_MAX) f[st.entries[i]] = i;
    return f;
}

static void access_cases() {
    // test_access.cpp: single element, permutation property, golden vectors
    CHECK(epoch_permutation(Seed{123}, 0, 1) == std::vector<uint32_t>{0});
    auto p = epoch_permutation(Seed{5}, 3, 10);
    std::sort(p.begin(), p.end());
    std::vector<uint32_t> iota10(10);
    std::iota(iota10.begin(), iota10.end(), 0u);
    CHECK(p == iota10);
    CHECK(epoch_permutation(Seed{42}, 0, 8) == golden("perm_seed42_epoch0_f8.txt"));
    CHECK(epoch_permutation(Seed{42}, 1, 8) == golden("perm_seed42_epoch1_f8.txt"));
    CHECK(epoch_permutation(Seed{42}, 0, 16) == golden("perm_seed42_epoch0_f16.txt"));
    // determinism and seed / epoch sensitivity
    CHECK(epoch_permutation(Seed{42}, 2, 100) == epoch_permutation(Seed{42}, 2, 100));
    CHECK(epoch_permutation(Seed{42}, 0, 100) != epoch_permutation(Seed{43}, 0, 100));
    CHECK(epoch_permutation(Seed{42}, 0, 100) != epoch_permutation(Seed{42}, 1, 100));
    // partition and coverage
    {
        PartitionSpec part{2, 2, 1, false};
        const auto s = build_access_streams(Seed{9}, 4, part);
        CHECK(s.size() == 2 && s[0].entries.size() == 2 && s[1].entries.size() == 2);
        std::set<uint32_t> all;
        for (const auto& st : s) all.insert(st.entries.begin(), st.entries.end());
        CHECK(all == (std::set<uint32_t>{0, 1, 2, 3}));
    }
    {
        PartitionSpec part{2, 2, 1, true};
        const auto s = build_access_streams(Seed{9}, 5, part);
        CHECK(s[0].entries.size() + s[1].entries.size() == 4);
    }
    {   // single worker = concatenated permutations, epoch offsets {0, 7, 14}
        PartitionSpec part{1, 3, 2, false};
        const auto s = build_access_streams(Seed{77}, 7, part);
        auto expect = epoch_permutation(Seed{77}, 0, 7);
        const auto e1 = epoch_permutation(Seed{77}, 1, 7);
        expect.insert(expect.end(), e1.begin(), e1.end());
        CHECK(s[0].entries == expect);
        CHECK(s[0].epoch_offsets == (std::vector<uint64_t>{0, 7, 14}));
    }
    {   // earlier epochs unchanged when the epoch count grows
        PartitionSpec p2{3, 6, 2, false}, p5 = p2;
        p5.epochs = 5;
        const auto s2 = build_access_streams(Seed{1}, 20, p2);
        const auto s5 = build_access_streams(Seed{1}, 20, p5);
        for (uint32_t w = 0; w < 3; ++w)
            CHECK(std::vector<uint32_t>(s5[w].entries.begin(),
                                        s5[w].entries.begin() + s2[w].entries.size()) == s2[w].entries);
    }
    {   // contiguous slices
        PartitionSpec part{2, 4, 1, true};
        const auto s = build_access_streams(Seed{5}, 8, part);
        const auto pm = epoch_permutation(Seed{5}, 0, 8);
        CHECK(s[0].entries == (std::vector<uint32_t>{pm[0], pm[1], pm[4], pm[5]}));
        CHECK(s[1].entries == (std::vector<uint32_t>{pm[2], pm[3], pm[6], pm[7]}));
    }
    {   // invalid partitions
        PartitionSpec part{2, 10, 1, true};
        CHECK_THROWS(build_access_streams(Seed{1}, 5, part));
        part.global_batch = 1;
        CHECK_THROWS(build_access_streams(Seed{1}, 5, part));
        CHECK_THROWS(epoch_permutation(Seed{1}, 0, 0));
    }
    {   // frequencies: conservation, single-worker degeneracy, worker_access_counts agreement
        const uint32_t F = 30, N = 3, E = 4;
        PartitionSpec part{N, 6, E, false};
        const auto s = build_access_streams(Seed{2}, F, part);
        PartitionSpec solo{1, 6, 3, false};
        const auto ss = build_access_streams(Seed{2}, F, solo);
        const auto sf = access_frequencies(ss[0], F, 0, 3);
        for (uint32_t k = 0; k < F; ++k) CHECK(sf.counts[k] == 3);
        std::vector<uint32_t> sum(F, 0);
        for (const auto& st : s) {
            const auto f = access_frequencies(st, F, 0, E);
            for (uint32_t k = 0; k < F; ++k) sum[k] += f.counts[k];
        }
        for (uint32_t k = 0; k < F; ++k) CHECK(sum[k] == E);
        for (uint32_t w = 0; w < N; ++w)
            CHECK(worker_access_counts(Seed{2}, F, part, w) == access_frequencies(s[w], F, 0, E).counts);
        const auto all = all_access_counts(Seed{2}, F, part);
        for (uint32_t w = 0; w < N; ++w) CHECK(all[w] == access_frequencies(s[w], F, 0, E).counts);
    }
    {   // epoch range selection
        PartitionSpec part{1, 4, 3, false};
        const auto s = build_access_streams(Seed{8}, 4, part);
        const auto f = access_frequencies(s[0], 4, 1, 2);
        for (uint32_t k = 0; k < 4; ++k) CHECK(f.counts[k] == 1);
    }
}

static void policy_cases() {
    {   // everything fits class 1 for a single worker
        const SystemConfig cfg = small_system(1, 1e6, 1e6);
        const auto ds = DatasetModel::generate(20, 1.0, 0, std::nullopt, 1);
        PartitionSpec part{1, 4, 2, false};
        const auto s = build_access_streams(Seed{1}, 20, part);
        const auto a = nopfs_assign_caches({access_frequencies(s[0], 20, 0, 2)}, cfg, ds, s);
        CHECK(a.class_lists[0][0].size() == 20 && a.class_lists[0][1].empty());
    }
    {   // greedy order puts the hot sample in the fast class (hand-built stream)
        const SystemConfig cfg = small_system(1, 1.0, 10.0);
        const auto ds = DatasetModel::from_sizes({1.0, 1.0});
        AccessStream st;
        st.entries = {0, 1, 0, 0, 1, 0, 0};
        st.epoch_offsets = {0, st.entries.size()};
        st.batch_offsets = {0, st.entries.size()};
        const auto a = nopfs_assign_caches({FrequencyTable{0, {5, 2}}}, cfg, ds, {st});
        CHECK(a.class_lists[0][0] == std::vector<uint32_t>{0});
        CHECK(a.class_lists[0][1] == std::vector<uint32_t>{1});
        CHECK(a.holders_of(0).size() == 1 && a.holders_of(0)[0].storage_class == 1);
    }
    {   // brute-force top-10 oracle (N=4, E=3, F=100, class 1 holds ten 1-MB samples)
        const uint32_t N = 4, E = 3, F = 100;
        const SystemConfig cfg = small_system(N, 10.0, 1e6);
        const auto ds = DatasetModel::generate(F, 1.0, 0, std::nullopt, 1);
        PartitionSpec part{N, 20, E, false};
        const auto s = build_access_streams(Seed{7}, F, part);
        std::vector<FrequencyTable> fr;
        for (const auto& st : s) fr.push_back(access_frequencies(st, F, 0, E));
        const auto a = nopfs_assign_caches(fr, cfg, ds, s);
        for (uint32_t w = 0; w < N; ++w) {
            const auto first = first_pos(s[w], F);
            std::vector<uint32_t> order;
            for (uint32_t k = 0; k < F; ++k)
                if (fr[w].counts[k] > 0) order.push_back(k);
            std::stable_sort(order.begin(), order.end(), [&](uint32_t x, uint32_t y) {
                if (fr[w].counts[x] != fr[w].counts[y]) return fr[w].counts[x] > fr[w].counts[y];
                return first[x] < first[y];
            });
            CHECK(std::set<uint32_t>(order.begin(), order.begin() + 10) ==
                  std::set<uint32_t>(a.class_lists[w][0].begin(), a.class_lists[w][0].end()));
            CHECK(a.class_lists[w][1].size() == order.size() - 10);
            for (size_t i = 1; i < a.class_lists[w][0].size(); ++i)
                CHECK(first[a.class_lists[w][0][i - 1]] < first[a.class_lists[w][0][i]]);
        }
    }
    {   // capacities respected, at most one class per sample, never-read samples unassigned
        const uint32_t N = 2, F = 60;
        const SystemConfig cfg = small_system(N, 7.5, 13.0);
        const auto ds = DatasetModel::generate(F, 1.0, 0.4, std::nullopt, 3);
        PartitionSpec part{N, 10, 4, false};
        const auto s = build_access_streams(Seed{11}, F, part);
        std::vector<FrequencyTable> fr;
        for (const auto& st : s) fr.push_back(access_frequencies(st, F, 0, 4));
        const auto a = nopfs_assign_caches(fr, cfg, ds, s);
        for (uint32_t w = 0; w < N; ++w) {
            std::set<uint32_t> seen;
            for (uint32_t j = 0; j < 2; ++j) {
                double bytes = 0;
                for (uint32_t k : a.class_lists[w][j]) {
                    bytes += ds.sizes_mb[k];
                    CHECK(seen.insert(k).second);
                    CHECK(fr[w].counts[k] > 0);
                }
                CHECK(bytes <= cfg.storage[j + 1].capacity_mb + 1e-9);
            }
        }
        // holder CSR consistent with the class lists; build_index reproduces it
        CacheAssignment b = a;
        b.build_index(F);
        CHECK(b.holder_offsets == a.holder_offsets);
        CHECK(b.holders.size() == a.holders.size());
        for (size_t i = 0; i < a.holders.size(); ++i)
            CHECK(b.holders[i].worker == a.holders[i].worker &&
                  b.holders[i].storage_class == a.holders[i].storage_class &&
                  b.holders[i].position == a.holders[i].position);
        for (uint32_t k = 0; k < F; ++k)
            for (const auto& h : a.holders_of(k))
                CHECK(a.class_lists[h.worker][h.storage_class - 1][h.position] == k);
    }
    {   // prefetch order is a subsequence of first-access order
        const SystemConfig cfg = small_system(2, 16.0, 8.0);
        const auto ds = DatasetModel::generate(24, 1.0, 0, std::nullopt, 1);
        PartitionSpec part{2, 4, 2, false};
        const auto s = build_access_streams(Seed{5}, 24, part);
        std::vector<FrequencyTable> fr;
        for (const auto& st : s) fr.push_back(access_frequencies(st, 24, 0, 2));
        const auto a = nopfs_assign_caches(fr, cfg, ds, s);
        for (uint32_t w = 0; w < 2; ++w) {
            const auto first = first_pos(s[w], 24);
            for (const auto& list : a.class_lists[w])
                for (size_t i = 1; i < list.size(); ++i) CHECK(first[list[i - 1]] < first[list[i]]);
        }
    }
}

int main() {
    try {
        access_cases();
        policy_cases();
    } catch (const std::exception& e) {
        std::fprintf(stderr, "exception: %s\n", e.what());
        return 2;
    }
    std::printf("compat_tests: %d checks, %d failures\n", g_checks, g_fail);
    return g_fail ? 1 : 0;
}
