// Drop-in implementation of the reference's hot-path C++ API (namespace clairsim) on top of
// the clairplan C ABI.  Compiled against the reference's own public headers
// (proj/include/clairsim/{access,policies}.hpp), so a clairsim build links this library in
// place of access.cpp and of the NoPFS part of policies.cpp.
//
// Every function keeps the reference signature, value semantics (host std::vector results
// owned by the caller) and error behaviour (std::invalid_argument with the same text).
// The work runs on the GPU selected by CLAIRPLAN_DEVICE (default 0); there is no CPU path.
#include <cstdlib>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../../include/clairplan.h"
#include "clairsim/access.hpp"
#include "clairsim/policies.hpp"

namespace clairsim {

namespace {

int device() {
    const char* e = std::getenv("CLAIRPLAN_DEVICE");
    return e ? std::atoi(e) : 0;
}

void check(int rc) {
    if (rc == CLAIRPLAN_OK) return;
    const std::string msg = clairplan_last_error();
    if (rc == CLAIRPLAN_EINVAL) throw std::invalid_argument(msg);
    throw std::runtime_error("clairplan error " + std::to_string(rc) + ": " + msg);
}

clairplan_config make_config(Seed seed, uint32_t samples, const PartitionSpec& part) {
    clairplan_config c{};
    c.seed = seed.value;
    c.samples = samples;
    c.num_workers = part.num_workers;
    c.global_batch = part.global_batch;
    c.epochs = part.epochs;
    c.drop_last = part.drop_last ? 1 : 0;
    c.device = device();
    return c;
}

// Epoch/batch offsets of worker w (pure functions of the partition, access.cpp:59-78).
void fill_offsets(AccessStream& st, uint32_t samples, const PartitionSpec& part) {
    const uint64_t B = part.global_batch;
    const uint64_t full = samples / B;
    const uint64_t tail = part.drop_last ? 0 : samples % B;
    st.epoch_offsets.assign(1, 0);
    st.batch_offsets.assign(1, 0);
    uint64_t pos = 0;
    for (uint32_t e = 0; e < part.epochs; ++e) {
        for (uint64_t h = 0; h < full + (tail > 0 ? 1 : 0); ++h) {
            const auto [b, en] = batch_slice(h < full ? B : tail, part.num_workers, st.worker_id);
            pos += en - b;
            st.batch_offsets.push_back(pos);
        }
        st.epoch_offsets.push_back(pos);
    }
}

}  // namespace

// access.cpp:33-39
std::pair<uint64_t, uint64_t> batch_slice(uint64_t batch_size, uint32_t workers, uint32_t worker) {
    const uint64_t base = batch_size / workers;
    const uint64_t extra = batch_size % workers;
    const uint64_t begin = worker * base + (worker < extra ? worker : extra);
    return {begin, begin + base + (worker < extra ? 1 : 0)};
}

// access.cpp:41-50 (messages come from the library, identical to the reference)
void PartitionSpec::validate(uint64_t samples) const {
    if (samples > 0xFFFFFFFFull) throw std::invalid_argument("dataset too large");
    clairplan_config c = make_config(Seed{0}, static_cast<uint32_t>(samples), *this);
    check(clairplan_validate(&c));
}

// access.hpp:58
std::vector<uint32_t> epoch_permutation(Seed seed, uint32_t epoch, uint32_t samples) {
    std::vector<uint32_t> out(samples);
    check(clairplan_epoch_permutation(seed.value, epoch, samples, out.data(), device()));
    return out;
}

// access.hpp:62-63
std::vector<AccessStream> build_access_streams(Seed seed, uint32_t samples,
                                               const PartitionSpec& part) {
    part.validate(samples);
    clairplan_config c = make_config(seed, samples, part);
    clairplan_t h = nullptr;
    check(clairplan_create(&c, &h));
    std::vector<AccessStream> streams(part.num_workers);
    try {
        check(clairplan_build(h));
        for (uint32_t w = 0; w < part.num_workers; ++w) {
            auto& st = streams[w];
            st.worker_id = w;
            const uint64_t n = clairplan_stream_offset(h, w + 1) - clairplan_stream_offset(h, w);
            st.entries.resize(n);
            uint64_t len = 0;
            check(clairplan_export_stream(h, w, st.entries.data(), n, &len));
            fill_offsets(st, samples, part);
        }
    } catch (...) {
        clairplan_destroy(h);
        throw;
    }
    clairplan_destroy(h);
    return streams;
}

// access.hpp:66-67
FrequencyTable access_frequencies(const AccessStream& stream, uint32_t samples,
                                  uint32_t epoch_begin, uint32_t epoch_end) {
    FrequencyTable t;
    t.worker_id = stream.worker_id;
    t.counts.assign(samples, 0);
    check(clairplan_access_frequencies(stream.entries.data(), stream.epoch_offsets.data(),
                                       stream.epoch_count(), samples, epoch_begin, epoch_end,
                                       t.counts.data(), device()));
    return t;
}

// access.hpp:71-72
std::vector<uint32_t> worker_access_counts(Seed seed, uint32_t samples, const PartitionSpec& part,
                                           uint32_t worker) {
    part.validate(samples);
    clairplan_config c = make_config(seed, samples, part);
    std::vector<uint32_t> out(samples);
    check(clairplan_worker_access_counts(&c, worker, out.data()));
    return out;
}

// access.hpp:76-77
std::vector<std::vector<uint32_t>> all_access_counts(Seed seed, uint32_t samples,
                                                     const PartitionSpec& part) {
    part.validate(samples);
    clairplan_config c = make_config(seed, samples, part);
    std::vector<uint32_t> flat(static_cast<size_t>(part.num_workers) * samples);
    check(clairplan_all_access_counts(&c, flat.data()));
    std::vector<std::vector<uint32_t>> out(part.num_workers);
    for (uint32_t w = 0; w < part.num_workers; ++w)
        out[w].assign(flat.begin() + static_cast<size_t>(w) * samples,
                      flat.begin() + static_cast<size_t>(w + 1) * samples);
    return out;
}

// policies.hpp:88-90 — explicit streams and frequency tables (any content, as the reference)
CacheAssignment nopfs_assign_caches(const std::vector<FrequencyTable>& freqs,
                                    const SystemConfig& cfg, const DatasetModel& dataset,
                                    const std::vector<AccessStream>& streams) {
    const uint32_t N = cfg.workers;
    const uint32_t J = cfg.cache_class_count();
    const uint32_t F = static_cast<uint32_t>(dataset.samples);
    CacheAssignment a;
    a.class_lists.assign(N, std::vector<std::vector<uint32_t>>(J));
    if (J == 0 || N == 0) {  // policies.cpp:151 loop does nothing; build_index over F
        a.build_index(dataset.samples);
        return a;
    }
    std::vector<uint64_t> offsets(N + 1, 0);
    for (uint32_t w = 0; w < N; ++w) offsets[w + 1] = offsets[w] + streams[w].entries.size();
    std::vector<uint32_t> entries(offsets[N]);
    for (uint32_t w = 0; w < N; ++w)
        std::copy(streams[w].entries.begin(), streams[w].entries.end(), entries.begin() + offsets[w]);
    std::vector<uint32_t> counts(static_cast<size_t>(N) * F);
    for (uint32_t w = 0; w < N; ++w)
        std::copy(freqs[w].counts.begin(), freqs[w].counts.end(),
                  counts.begin() + static_cast<size_t>(w) * F);
    std::vector<double> caps(J);
    for (uint32_t j = 0; j < J; ++j) caps[j] = cfg.storage[j + 1].capacity_mb;
    clairplan_t h = nullptr;
    check(clairplan_assign_from_streams(N, F, entries.data(), offsets.data(), counts.data(), J,
                                        caps.data(), dataset.sizes_mb.data(), device(), &h));
    try {
        std::vector<uint64_t> off(static_cast<size_t>(N) * J), len(static_cast<size_t>(N) * J);
        check(clairplan_class_list_bounds(h, off.data(), len.data()));
        uint64_t total = 0;
        for (uint64_t x : len) total += x;
        std::vector<uint32_t> flat(total);
        check(clairplan_export_class_lists(h, flat.data(), total));
        uint64_t o = 0;
        for (uint32_t w = 0; w < N; ++w)
            for (uint32_t j = 0; j < J; ++j) {
                const uint64_t n = len[static_cast<size_t>(w) * J + j];
                a.class_lists[w][j].assign(flat.begin() + o, flat.begin() + o + n);
                o += n;
            }
        const uint64_t* dho = nullptr;
        const uint32_t* dh = nullptr;
        uint64_t H = 0;
        check(clairplan_device_holders(h, &dho, &dh, &H));
        if (H > 0xFFFFFFFFull)
            throw std::overflow_error("EOVERFLOW: holder count exceeds the u32 holder_offsets");
        std::vector<uint64_t> ho(F + 1);
        std::vector<uint32_t> hv(3 * H);
        check(clairplan_export_holders(h, ho.data(), hv.data(), H));
        a.holder_offsets.resize(F + 1);
        for (uint32_t k = 0; k <= F; ++k) a.holder_offsets[k] = static_cast<uint32_t>(ho[k]);
        a.holders.resize(H);
        for (uint64_t i = 0; i < H; ++i)
            a.holders[i] = CacheAssignment::Holder{hv[3 * i], hv[3 * i + 1], hv[3 * i + 2]};
    } catch (...) {
        clairplan_destroy(h);
        throw;
    }
    clairplan_destroy(h);
    return a;
}

// policies.cpp:124-142 — rebuilds the CSR on the GPU from the (possibly edited) class lists
void CacheAssignment::build_index(uint64_t samples) {
    const uint32_t N = static_cast<uint32_t>(class_lists.size());
    const uint32_t J = N ? static_cast<uint32_t>(class_lists[0].size()) : 0;
    std::vector<uint64_t> off(static_cast<size_t>(N) * J + 1, 0);
    for (uint32_t w = 0; w < N; ++w)
        for (uint32_t j = 0; j < J; ++j)
            off[static_cast<size_t>(w) * J + j + 1] =
                off[static_cast<size_t>(w) * J + j] + class_lists[w][j].size();
    std::vector<uint32_t> flat(off.back());
    for (uint32_t w = 0; w < N; ++w)
        for (uint32_t j = 0; j < J; ++j)
            std::copy(class_lists[w][j].begin(), class_lists[w][j].end(),
                      flat.begin() + off[static_cast<size_t>(w) * J + j]);
    // the reference's u32 holder_offsets (policies.hpp:59) cannot hold 2^32 or more holders:
    // refuse (EOVERFLOW) instead of truncating; clairplan_build_index keeps u64 offsets
    if (flat.size() > 0xFFFFFFFFull)
        throw std::overflow_error("EOVERFLOW: " + std::to_string(flat.size()) +
                                  " holders exceed the u32 holder_offsets of CacheAssignment");
    std::vector<uint64_t> ho(samples + 1);
    std::vector<uint32_t> hv(3 * flat.size() + 3);
    check(clairplan_build_index(N, J, samples, flat.data(), off.data(), ho.data(), hv.data(),
                                device()));
    holder_offsets.resize(samples + 1);
    for (uint64_t k = 0; k <= samples; ++k) holder_offsets[k] = static_cast<uint32_t>(ho[k]);
    holders.resize(flat.size());
    for (size_t i = 0; i < flat.size(); ++i)
        holders[i] = Holder{hv[3 * i], hv[3 * i + 1], hv[3 * i + 2]};
}

}  // namespace clairsim
