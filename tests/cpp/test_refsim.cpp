// TEST INFRASTRUCTURE: the reference's own build_policy / simulate (policies.cpp:446-456,
// simulator.cpp:393-399), compiled unmodified into oracle/_ref/libclairsim_sim.so, driving
// the planner through ordinary dynamic-symbol resolution.
//
// Built twice from this file (tests/cpp/Makefile):
//   refsim_cpu   links libclairsim_sim.so only: the all-CPU reference
//   refsim_b200  links libclairsim_b200.so first: its clairsim::build_access_streams /
//                nopfs_assign_caches / ... definitions take precedence over the reference
//                library's own for every call, including the calls inside the reference's
//                build_policy (interposable default-visibility symbols, -fPIC)
// Both print the same digest when the drop-in is exact; pytest -m gpu compares them.
#include <dlfcn.h>

#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "clairsim/access.hpp"
#include "clairsim/policies.hpp"
#include "clairsim/scenarios.hpp"
#include "clairsim/simulator.hpp"

using namespace clairsim;

namespace {

struct Digest {
    uint64_t h = 1469598103934665603ull;
    void add(const void* p, size_t n) {
        const unsigned char* c = static_cast<const unsigned char*>(p);
        for (size_t i = 0; i < n; ++i) h = (h ^ c[i]) * 1099511628211ull;
    }
    template <typename T>
    void vec(const std::vector<T>& v) {
        const uint64_t n = v.size();
        add(&n, sizeof n);
        if (n) add(v.data(), n * sizeof(T));
    }
};

const char* owner_of(const void* fn) {
    Dl_info info;
    if (dladdr(fn, &info) && info.dli_fname) {
        const char* s = strrchr(info.dli_fname, '/');
        return s ? s + 1 : info.dli_fname;
    }
    return "?";
}

}  // namespace

int main(int argc, char** argv) {
    const std::string name = argc > 1 ? argv[1] : "imagenet1k";
    const double scale = argc > 2 ? std::stod(argv[2]) : 0.01;
    const uint32_t epochs = argc > 3 ? static_cast<uint32_t>(std::stoul(argv[3])) : 4;
    Scenario sc = make_scenario(name);
    scale_scenario(sc, scale);
    const DatasetModel dataset = sc.make_dataset(1);
    const PartitionSpec part{sc.system.workers, sc.global_batch(), epochs, true};
    const std::vector<AccessStream> streams =
        build_access_streams(Seed{42}, static_cast<uint32_t>(sc.samples), part);
    PolicySpec spec;
    spec.kind = PolicyKind::Nopfs;
    const BuiltPolicy policy = build_policy(spec, streams, sc.system, dataset);
    const SimResult r = simulate(sc.system, dataset, streams, policy);

    Digest ds, da, dr;
    for (const auto& s : streams) {
        ds.vec(s.entries);
        ds.vec(s.epoch_offsets);
        ds.vec(s.batch_offsets);
    }
    for (const auto& w : policy.assignment.class_lists)
        for (const auto& l : w) da.vec(l);
    da.vec(policy.assignment.holder_offsets);
    for (const auto& h : policy.assignment.holders) {
        da.add(&h.worker, 4);
        da.add(&h.storage_class, 4);
        da.add(&h.position, 4);
    }
    dr.add(&r.total_time_s, 8);
    dr.add(&r.stall_time_s, 8);
    dr.add(&r.perfect_bound_s, 8);
    dr.vec(r.worker_total_s);
    dr.vec(r.worker_stall_s);
    for (const auto& kv : r.demand) {
        dr.add(kv.first.data(), kv.first.size());
        dr.add(&kv.second.fetch_s, 8);
        dr.add(&kv.second.bytes_mb, 8);
    }
    for (const auto& e : r.epochs) dr.add(&e.time_s, 8);
    uint64_t holders = policy.assignment.holders.size();
    std::printf("planner build_access_streams=%s nopfs_assign_caches=%s\n",
                owner_of(reinterpret_cast<const void*>(&build_access_streams)),
                owner_of(reinterpret_cast<const void*>(&nopfs_assign_caches)));
    std::printf("scenario %s x%g F=%llu N=%u E=%u holders=%llu\n", name.c_str(), scale,
                (unsigned long long)sc.samples, sc.system.workers, epochs,
                (unsigned long long)holders);
    std::printf("digest streams=%016llx assignment=%016llx simulate=%016llx total_time=%a stall=%a\n",
                (unsigned long long)ds.h, (unsigned long long)da.h, (unsigned long long)dr.h,
                r.total_time_s, r.stall_time_s);
    return 0;
}
