"""GPU parity: the CUDA path (through the C ABI) against the reference / the oracle.

Bit-exact for everything: permutations, streams, tier assignments, prefetch orders, holder
CSR (integer/index work plus an order-sensitive double chain reproduced exactly)."""
import os

import numpy as np
import pytest

from _oracle import Plan as OPlan
from _oracle import plans_equal

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def cp():
    from paper_2101_08734_b200 import clairplan
    return clairplan


def device_plan(cp, seed, F, N, B, E, dl, caps, sizes):
    p = cp.Plan(seed, F, cp.PartitionSpec(N, B, E, dl), caps, sizes).build()
    offs, hold = p.holders()
    out = OPlan(N, len(caps), [p.stream(w) for w in range(N)], p.class_lists(), offs, hold)
    out.stats = p.stats()
    out.launches = p.launch_count()
    p.close()
    return out


def load_perm(name):
    with open(os.path.join(HERE, "golden", name)) as f:
        return np.array(f.read().split(), np.uint32)


def test_perm_golden(cp):
    assert np.array_equal(cp.epoch_permutation(42, 0, 8), load_perm("perm_seed42_epoch0_f8.txt"))
    assert np.array_equal(cp.epoch_permutation(42, 1, 8), load_perm("perm_seed42_epoch1_f8.txt"))
    assert np.array_equal(cp.epoch_permutation(42, 0, 16), load_perm("perm_seed42_epoch0_f16.txt"))
    assert list(cp.epoch_permutation(123, 0, 1)) == [0]
    with pytest.raises(ValueError, match="permutation needs samples >= 1"):
        cp.epoch_permutation(1, 0, 0)


def test_perm_random_small(cp, port):
    rng = np.random.default_rng(2)
    for _ in range(150):
        F = int(rng.integers(1, 5000))
        seed = int(rng.integers(0, 2**63))
        e = int(rng.integers(0, 1000))
        assert np.array_equal(cp.epoch_permutation(seed, e, F), port.epoch_permutation(seed, e, F)), \
            (seed, e, F)


@pytest.mark.parametrize("F,epoch", [(1_281_167, 0), (1_281_167, 89), (262_144, 7),
                                     (14_197_122, 3)])
def test_perm_large(cp, ref, F, epoch):
    assert np.array_equal(cp.epoch_permutation(42, epoch, F), ref.epoch_permutation(42, epoch, F))


CASES = [
    (42, 2000, 4, 128, 10, True, [20.0, 900.0], (0.1077, 0.1)),
    (7, 1500, 3, 7, 5, False, [5.0, 30.0], (0.1, 0.3)),
    (9, 1000, 16, 16, 6, True, [1e6, 1e6], (1.0, 0.0)),
    (1, 777, 5, 13, 4, False, [3.0], (0.5, 0.5)),
    (3, 600, 2, 9, 3, True, [2.0, 3.0, 40.0], (0.2, 0.1)),
    (11, 500, 4, 4, 20, True, [], (0.1, 0.1)),
    (5, 24, 2, 4, 2, False, [16.0, 8.0], (1.0, 0.0)),      # test_policies.cpp:328-350 shape
    (7, 100, 4, 20, 3, False, [10.0, 1e6], (1.0, 0.0)),    # test_policies.cpp:69-102 shape
    (11, 60, 2, 10, 4, False, [7.5, 13.0], (1.0, 0.4)),    # test_policies.cpp:104-125 shape
    (2, 30, 3, 6, 4, False, [5.0, 5.0], (1.0, 0.0)),
    (77, 7, 1, 3, 2, False, [100.0], (1.0, 0.0)),
    (13, 5000, 7, 300, 33, True, [25.0, 120.0], (0.1077, 0.2)),
    (21, 4096, 64, 64, 40, False, [3.0, 9.0], (0.1, 0.05)),
    (8, 3000, 5, 5, 300, True, [40.0, 400.0], (0.1, 0.1)),   # E > 255: two radix digits
    (17, 3000, 6, 60, 12, True, [2.0, 3.0, 5.0, 8.0], (0.1, 0.1)),              # J = 4: 3 planes
    (19, 2500, 9, 45, 15, False, [1.0, 2.0, 1.5, 4.0, 3.0, 9.0, 2.5], (0.2, 0.1)),  # J = 7
]


@pytest.mark.parametrize("case", CASES)
def test_plan_small_matches_reference(cp, ref, case):
    seed, F, N, B, E, dl, caps, (mu, sd) = case
    sizes = ref.generate_sizes(F, mu, sd, None, 1)
    a = ref.plan(seed, F, N, B, E, dl, caps, sizes)
    b = device_plan(cp, seed, F, N, B, E, dl, caps, sizes)
    assert plans_equal(a, b) is None


@pytest.mark.parametrize("case", [
    (4, 2000, 64, 64, 200, False, [30.0, 60.0], (0.1, 0.1)),   # >32 repeated workers: hash fallback
    (6, 6000, 3000, 3000, 3, True, [2.0, 5.0], (0.1, 0.1)),    # >2048 workers: v1 pipeline
])
def test_plan_fallback_paths(cp, ref, case):
    seed, F, N, B, E, dl, caps, (mu, sd) = case
    sizes = ref.generate_sizes(F, mu, sd, None, 1)
    a = ref.plan(seed, F, N, B, E, dl, caps, sizes)
    b = device_plan(cp, seed, F, N, B, E, dl, caps, sizes)
    assert plans_equal(a, b) is None


@pytest.mark.parametrize("case", CASES[:6])
def test_plan_v1_pipeline_matches_reference(cp, ref, case, monkeypatch):
    monkeypatch.setenv("CLAIRPLAN_FORCE_V1", "1")
    seed, F, N, B, E, dl, caps, (mu, sd) = case
    sizes = ref.generate_sizes(F, mu, sd, None, 1)
    a = ref.plan(seed, F, N, B, E, dl, caps, sizes)
    b = device_plan(cp, seed, F, N, B, E, dl, caps, sizes)
    assert plans_equal(a, b) is None


@pytest.mark.parametrize("case", CASES[:5] + [CASES[11]])
def test_linked_list_shuffle_fallback(cp, ref, case, monkeypatch):
    """The linked-list shuffle (perm.cu), the fallback after a bucket-region overflow of the
    contiguous-bucket shuffle (perm_fyc.cu), forced: plans and permutations equal the
    reference's."""
    monkeypatch.setenv("CLAIRPLAN_FY_LISTS", "1")
    seed, F, N, B, E, dl, caps, (mu, sd) = case
    sizes = ref.generate_sizes(F, mu, sd, None, 1)
    a = ref.plan(seed, F, N, B, E, dl, caps, sizes)
    b = device_plan(cp, seed, F, N, B, E, dl, caps, sizes)
    assert plans_equal(a, b) is None
    for F2, e in ((1_281_167, 3), (14_197_122, 1), (7, 0)):
        assert np.array_equal(cp.epoch_permutation(42, e, F2), ref.epoch_permutation(42, e, F2))


def test_plan_random_configs(cp, ref):
    rng = np.random.default_rng(9)
    for _ in range(25):
        F = int(rng.integers(10, 4000))
        N = int(rng.integers(1, 40))
        B = int(rng.integers(N, min(F, 8 * N + 30) + 1))
        E = int(rng.integers(1, 50))
        dl = bool(rng.integers(0, 2))
        J = int(rng.integers(0, 4))
        caps = [float(x) for x in rng.uniform(0.5, 200.0, J)]
        sizes = rng.uniform(0.001, 2.0, F) if rng.integers(0, 2) else np.full(F, 0.37)
        seed = int(rng.integers(0, 2**62))
        a = ref.plan(seed, F, N, B, E, dl, caps, sizes)
        b = device_plan(cp, seed, F, N, B, E, dl, caps, sizes)
        assert plans_equal(a, b) is None, (seed, F, N, B, E, dl, caps)


def config_sizes(ref, which):
    if which in (1, 2):
        return ref.generate_sizes(1_281_167, 0.1077, 0.1, 135_000.0, 1)
    if which == 3:
        return ref.generate_sizes(262_144, 16.0, 0.0, None, 1)
    raise ValueError(which)


def test_config1_imagenet1k_e10_n4(cp, ref):
    sizes = config_sizes(ref, 1)
    a = ref.plan(42, 1_281_167, 4, 128, 10, True, [120_000.0, 900_000.0], sizes)
    b = device_plan(cp, 42, 1_281_167, 4, 128, 10, True, [120_000.0, 900_000.0], sizes)
    assert plans_equal(a, b) is None
    assert b.stats["accesses"] == 12_811_520 and b.stats["pairs"] == 4_836_013


def test_config3_cosmoflow_e100_n1024(cp, ref):
    sizes = config_sizes(ref, 3)
    a = ref.plan(42, 262_144, 1024, 16 * 1024, 100, True, [120_000.0, 900_000.0], sizes)
    b = device_plan(cp, 42, 262_144, 1024, 16 * 1024, 100, True, [120_000.0, 900_000.0], sizes)
    assert plans_equal(a, b) is None
    assert b.stats["pairs"] == 24_985_949


def test_config2_imagenet1k_e90_n256(cp, ref):
    sizes = config_sizes(ref, 2)
    a = ref.plan(42, 1_281_167, 256, 32 * 256, 90, True, [120_000.0, 900_000.0], sizes,
                 mode=1, threads=os.cpu_count() or 4)
    b = device_plan(cp, 42, 1_281_167, 256, 32 * 256, 90, True, [120_000.0, 900_000.0], sizes)
    assert plans_equal(a, b) is None
    assert b.stats["accesses"] == 115_015_680 and b.stats["pairs"] == 97_174_801
    assert b.stats["path"] == "allfit"  # the benchmarked pipeline


ALLFIT_CASES = [
    (42, 2000, 4, 128, 10, True, [1e6, 1e6], (0.1077, 0.1)),
    (9, 1000, 16, 16, 6, True, [1e6, 1e6], (1.0, 0.0)),
    (7, 1500, 3, 7, 5, False, [1e5], (0.1, 0.3)),
    (13, 5000, 7, 300, 33, True, [1e4, 1.0, 5.0], (0.1077, 0.2)),
    (77, 7, 1, 3, 2, False, [100.0], (1.0, 0.0)),
    (8, 3000, 5, 5, 300, True, [1e6, 2.0], (0.1, 0.1)),
]


@pytest.mark.parametrize("case", ALLFIT_CASES)
def test_allfit_path_matches_reference(cp, ref, case, monkeypatch):
    """Every worker provably fits class 1: the all-fit pipeline (no tier order) and the full
    tier-order pipeline both equal the reference."""
    seed, F, N, B, E, dl, caps, (mu, sd) = case
    sizes = ref.generate_sizes(F, mu, sd, None, 1)
    a = ref.plan(seed, F, N, B, E, dl, caps, sizes)
    b = device_plan(cp, seed, F, N, B, E, dl, caps, sizes)
    # the worker sums come from the tile sample pass (E <= 128); the lane fallback takes the
    # tier path
    assert b.stats["path"] == ("allfit" if E <= 128 else "tier")
    assert plans_equal(a, b) is None
    monkeypatch.setenv("CLAIRPLAN_NO_ALLFIT", "1")
    c = device_plan(cp, seed, F, N, B, E, dl, caps, sizes)
    assert c.stats["path"] == "tier"
    assert plans_equal(a, c) is None


def test_allfit_capacity_boundary(cp, ref):
    """Class-1 capacity at, just below and just above the largest per-worker candidate sum:
    whichever pipeline the fit test picks, the plan equals the reference."""
    seed, F, N, B, E = 4, 3000, 6, 60, 8
    sizes = ref.generate_sizes(F, 0.3, 0.2, None, 1)
    b0 = device_plan(cp, seed, F, N, B, E, True, [1e9], sizes)
    sums = [float(np.sum(sizes[np.unique(s)])) for s in b0.streams]
    top = max(sums)
    paths = set()
    for C in (top, np.nextafter(top, 0), np.nextafter(top, np.inf), top * (1 - 1e-9),
              top * (1 + 1e-9), top * (1 + 1e-6), top * (1 + 1e-3), min(sums), 0.5 * top):
        a = ref.plan(seed, F, N, B, E, True, [float(C), 5.0], sizes)
        b = device_plan(cp, seed, F, N, B, E, True, [float(C), 5.0], sizes)
        paths.add(b.stats["path"])
        assert plans_equal(a, b) is None, C
    assert paths == {"allfit", "tier"}


def test_reassign_after_allfit_build(cp, ref):
    F, N, B, E = 20_000, 8, 256, 12
    sizes = ref.generate_sizes(F, 0.1077, 0.2, None, 1)
    p = cp.Plan(3, F, cp.PartitionSpec(N, B, E, True), [1e7, 1e7], sizes).build()
    assert p.stats()["path"] == "allfit"
    for caps in ([30.0, 60.0], [1e7, 1e7], [0.05, 0.2]):
        p.reassign(caps)
        offs, hold = p.holders()
        got = OPlan(N, 2, [p.stream(w) for w in range(N)], p.class_lists(), offs, hold)
        want = ref.plan(3, F, N, B, E, True, caps, sizes)
        assert plans_equal(want, got) is None, caps
    p.close()


def test_generic_assign_matches_reference(cp, ref):
    # test_policies.cpp:54-67
    st = cp.AccessStream(0, np.array([0, 1, 0, 0, 1, 0, 0], np.uint32))
    a = cp.nopfs_assign_caches([cp.FrequencyTable(0, np.array([5, 2], np.uint32))], [1.0, 10.0],
                               [1.0, 1.0], [st])
    assert list(a.class_lists[0][0]) == [0] and list(a.class_lists[0][1]) == [1]
    rng = np.random.default_rng(5)
    for _ in range(20):
        N, F = int(rng.integers(1, 5)), int(rng.integers(5, 60))
        streams = [rng.integers(0, F, int(rng.integers(0, 80))).astype(np.uint32) for _ in range(N)]
        counts = rng.integers(0, 4, (N, F)).astype(np.uint32)
        sizes = rng.uniform(0.1, 2.0, F)
        caps = [float(rng.uniform(1, 10)), float(rng.uniform(1, 30))]
        r = ref.assign_from_streams(streams, counts, caps, sizes)
        g = cp.nopfs_assign_caches([cp.FrequencyTable(w, counts[w]) for w in range(N)], caps, sizes,
                                   [cp.AccessStream(w, streams[w]) for w in range(N)])
        got = OPlan(N, 2, streams, g.class_lists, g.holder_offsets, g.holders)
        assert plans_equal(r, got, check_streams=False) is None


def test_reassign_matches_fresh_plans(cp, ref):
    """Capacity sweep: one build, then reassign per grid point == a fresh
    reference plan with those capacities."""
    F, N, B, E = 20_000, 8, 256, 12
    sizes = ref.generate_sizes(F, 0.1077, 0.2, None, 1)
    p = cp.Plan(11, F, cp.PartitionSpec(N, B, E, True), [100.0, 400.0], sizes).build()
    for caps in ([100.0, 400.0], [30.0, 60.0], [1e6, 1.0], [0.05, 0.2], [250.0, 90.0]):
        p.reassign(caps)
        offs, hold = p.holders()
        got = OPlan(N, 2, [p.stream(w) for w in range(N)], p.class_lists(), offs, hold)
        want = ref.plan(11, F, N, B, E, True, caps, sizes)
        assert plans_equal(want, got) is None, caps
    p.close()


def test_build_index_matches_device_csr(cp, ref):
    sizes = ref.generate_sizes(3000, 0.1, 0.1, None, 1)
    p = cp.Plan(5, 3000, cp.PartitionSpec(6, 60, 12, True), [30.0, 100.0], sizes).build()
    a = p.assignment()
    p.close()
    b = cp.CacheAssignment(a.class_lists)
    b.build_index(3000)
    assert np.array_equal(a.holder_offsets, b.holder_offsets)
    assert np.array_equal(a.holders, b.holders)


def test_counts_entry_points(cp, ref):
    F, N, B, E = 30, 3, 6, 4
    part = cp.PartitionSpec(N, B, E, False)
    # test_access.cpp:107-131: conservation and worker_access_counts == access_frequencies
    streams = cp.build_access_streams(2, F, part)
    rp = ref.plan(2, F, N, B, E, False, [], np.ones(F), keep=True)
    for w in range(N):
        assert np.array_equal(streams[w].entries, rp.streams[w])
        assert np.array_equal(streams[w].epoch_offsets, rp.epoch_offsets[w])
        assert np.array_equal(streams[w].batch_offsets, rp.batch_offsets[w])
        for eb, ee in ((0, E), (1, 3), (2, 2), (0, E + 3)):
            f = cp.access_frequencies(streams[w], F, eb, ee)
            assert np.array_equal(f.counts, ref.access_frequencies(rp, w, eb, ee, F))
        assert np.array_equal(cp.worker_access_counts(2, F, part, w),
                              ref.worker_access_counts(2, F, N, B, E, False, w))
    ref.free(rp)
    allc = cp.all_access_counts(2, F, part)
    assert np.array_equal(allc, ref.all_access_counts(2, F, N, B, E, False))
    assert np.all(allc.sum(axis=0) == E)
    # acceptance.cpp:102-107 shape (Lemma-1 suite input): B = N, no drop
    for N in (2, 4, 16):
        p = cp.PartitionSpec(N, N, 10, False)
        assert np.array_equal(cp.all_access_counts(3, 1000, p),
                              ref.all_access_counts(3, 1000, N, N, 10, False))


def test_rebuild_is_deterministic(cp, ref):
    sizes = ref.generate_sizes(3000, 0.1, 0.1, None, 1)
    p = cp.Plan(5, 3000, cp.PartitionSpec(6, 60, 12, True), [30.0, 100.0], sizes)
    p.build()
    s1, c1, h1 = p.streams_flat(), p.class_lists(), p.holders()
    p.build()
    s2, c2, h2 = p.streams_flat(), p.class_lists(), p.holders()
    assert np.array_equal(s1, s2)
    assert all(np.array_equal(x, y) for a, b in zip(c1, c2) for x, y in zip(a, b))
    assert np.array_equal(h1[0], h2[0]) and np.array_equal(h1[1], h2[1])
    p.close()


def test_cpp_compat_suite():
    """Reference test cases re-hosted in C++ against libclairsim_b200.so (the drop-in)."""
    import subprocess
    exe = os.path.join(HERE, "cpp", "compat_tests")
    if not os.path.exists(exe):
        pytest.skip("compat_tests not built (needs the reference headers at build time)")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failures" in r.stdout


@pytest.mark.parametrize("preset", [("imagenet1k", "0.01", "4"), ("cosmoflow", "0.02", "3"),
                                    ("imagenet22k", "0.001", "3")])
def test_reference_simulator_over_the_dropin(preset):
    """The reference's own build_policy(Nopfs) + simulate (policies.cpp:446-456,
    simulator.cpp:393-399), compiled unmodified into oracle/_ref/libclairsim_sim.so, with
    libclairsim_b200.so linked ahead of it (tests/cpp/Makefile): every planner call, also
    the ones made inside the reference library, resolves to the drop-in; streams, cache
    assignment, holder CSR and the simulation result digest equal the all-CPU build's."""
    import subprocess
    exe = {n: os.path.join(HERE, "cpp", n) for n in ("refsim_cpu", "refsim_b200")}
    if not all(os.path.exists(x) for x in exe.values()):
        pytest.skip("refsim drivers not built (need the reference sources at build time)")
    out = {}
    for n, x in exe.items():
        r = subprocess.run([x, *preset], capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stdout + r.stderr
        out[n] = r.stdout.splitlines()
    assert "nopfs_assign_caches=libclairsim_b200.so" in out["refsim_b200"][0]
    assert "build_access_streams=libclairsim_b200.so" in out["refsim_b200"][0]
    assert "nopfs_assign_caches=libclairsim_sim.so" in out["refsim_cpu"][0]
    assert out["refsim_cpu"][1:] == out["refsim_b200"][1:], (out["refsim_cpu"], out["refsim_b200"])


def test_choose_sources_match_reference(cp, ref):
    """The plan consumer: the device's batched source chooser equals the
    reference's choose_source (policies.cpp:184-233) query by query — local / remote /
    PFS, progress thresholds, heuristic mode, the allow flags, ties (Local = Remote unit times
    on the preset system) broken Local > Remote > lowest worker."""
    F, N, B, E = 20_000, 8, 256, 6
    for caps in ([150.0, 400.0], [1e6, 1e6], [20.0, 60.0, 100.0]):
        sizes = ref.generate_sizes(F, 0.1077, 0.2, None, 1)
        rp = ref.plan(42, F, N, B, E, True, caps, sizes, keep=True)
        p = cp.Plan(42, F, cp.PartitionSpec(N, B, E, True), caps, sizes).build()
        J = len(caps)
        rng = np.random.default_rng(len(caps))
        lens = np.array([[len(rp.class_lists[w][j]) for j in range(J)] for w in range(N)], np.uint64)
        nq = 30_000
        samples = rng.integers(0, F, nq).astype(np.uint32)
        workers = rng.integers(0, N, nq).astype(np.uint32)
        for trial in range(6):
            frac = rng.uniform(0, 1.2, (N, J))
            progress = np.minimum((lens * frac).astype(np.uint64), lens)
            if trial == 0:
                progress = lens.copy()        # every prefetch done
            gamma = int(rng.integers(1, 9))
            heuristic = bool(trial % 2)
            al, ar = (True, True) if trial < 4 else ((trial == 4), (trial == 5))
            lt, rt, pf = ref.unit_times(N, caps, gamma)
            want = ref.choose_sources(rp, N, caps, progress, gamma, samples, workers, al, ar, heuristic)
            got = p.choose_sources(samples, workers, progress, lt, rt, pf, al, ar, heuristic)
            assert np.array_equal(got["kind"], want[:, 0].astype(np.uint8)), (caps, trial)
            assert np.array_equal(got["storage_class"], want[:, 1].astype(np.uint8)), (caps, trial)
            assert np.array_equal(got["worker"], want[:, 2]), (caps, trial)
            kinds = set(np.unique(got["kind"]).tolist())
            if trial == 0 and al and ar:
                assert cp.SRC_LOCAL in kinds and cp.SRC_REMOTE in kinds
        # the "earliest remote holder" table against a restatement over the holder CSR
        lt, rt, pf = ref.unit_times(N, caps, 1)
        eh = p.earliest_holders(rt)
        offs, hold = p.holders()
        for k in rng.integers(0, F, 2000):
            hs = hold[offs[k]:offs[k + 1]]
            if len(hs) == 0:
                assert list(eh[k]) == [0xFFFFFFFF] * 3
                continue
            best = min(hs.tolist(), key=lambda h: (rt[h[1] - 1], h[2], h[0]))
            assert list(eh[k]) == best, k
        ref.free(rp)
        p.close()


def test_analysis_reuse_monte_carlo_c1(cp, ref):
    """Acceptance C1 (acceptance.cpp:76-93) on device counts: monte_carlo_histogram
    (analysis.cpp:84-96) equals the reference's bucket for bucket, and its hot count lies
    within 5% of the analytic expectation (expected_hot_samples, ~31,635)."""
    N, E, F, delta = 16, 90, 1_281_167, 0.8
    got = cp.monte_carlo_histogram(1, N, E, F)
    want = ref.monte_carlo_histogram(1, N, E, F)
    assert np.array_equal(got, want)
    assert int(got.sum()) == F
    expected = ref.expected_hot_samples(N, E, F, delta)
    assert abs(expected - 31634.685810763236) < 1e-6
    hot = int(got[ref.hot_count_threshold(N, E, delta):].sum())
    assert abs(hot - expected) / expected < 0.05
    for seed, N, E, F in ((3, 4, 10, 5000), (7, 16, 100, 20_011)):
        assert np.array_equal(cp.monte_carlo_histogram(seed, N, E, F),
                              ref.monte_carlo_histogram(seed, N, E, F))


def test_analysis_reuse_lemma1_c2(cp, ref):
    """Acceptance C2 (acceptance.cpp:98-158): the Lemma-1 counterpart bounds over 50 seeds,
    N in {2, 4, 16}, E in {4, 10, 90}, F in {1e3, 1e4}, evaluated from device per-sample count
    extremes (after removing one worker holding the maximum, the others' minimum is the
    minimum, and symmetrically); extremes equal the reference's all_access_counts reductions."""
    checked = 0
    for N in (2, 4, 16):
        for E in (4, 10, 90):
            for F in (1000, 10000):
                part = cp.PartitionSpec(N, N, E, False)
                for seed in range(50):
                    hi, lo = cp.count_extremes(seed, F, part)
                    if seed % 17 == 0:
                        allc = ref.all_access_counts(seed, F, N, N, E, False)
                        assert np.array_equal(hi, allc.max(axis=0)) and np.array_equal(lo, allc.min(axis=0))
                    for delta in (0.2, 0.4, 0.6, 0.8, 1.0):
                        if delta > N - 1:
                            continue
                        hth, clow, lth, chigh = ref.lemma1_bounds(N, E, delta)
                        assert not np.any((hi >= hth) & (lo > clow)), (N, E, F, seed, delta)
                        assert not np.any((lo.astype(np.int64) <= lth) & (hi < chigh)), (N, E, F, seed, delta)
                        checked += F
    assert checked > 0


def test_wire_image_round_trip_and_shard_merge(cp, ref):
    """Plan wire format: the device writer's image parses with every section
    checksum verified and equals the plan's exports and the reference; images of three
    worker-range handles merged on the host equal the single-handle plan."""
    from paper_2101_08734_b200 import wire
    F, N, B, E = 30_000, 12, 240, 9
    for caps in ([20.0, 60.0], [1e6, 1e6]):
        sizes = ref.generate_sizes(F, 0.1077, 0.2, None, 1)
        p = cp.Plan(5, F, cp.PartitionSpec(N, B, E, True), caps, sizes).build()
        img = wire.parse(p.wire())
        want = ref.plan(5, F, N, B, E, True, caps, sizes)
        assert np.array_equal(img["streams"], np.concatenate(want.streams))
        assert all(np.array_equal(x, y) for a, b in zip(wire.class_lists(img), want.class_lists)
                   for x, y in zip(a, b))
        assert np.array_equal(img["holder_offsets"], want.holder_offsets.astype(np.uint64))
        assert np.array_equal(img["holders"], want.holders)
        assert list(img["capacities"]) == caps
        p.close()
        shards = []
        for wr in ((0, 5), (5, 6), (6, 12)):
            q = cp.Plan(5, F, cp.PartitionSpec(N, B, E, True), caps, sizes, worker_range=wr).build()
            shards.append(wire.parse(q.wire()))
            q.close()
        m = wire.merge_shards(shards[::-1])
        assert np.array_equal(m["streams"], img["streams"])
        assert np.array_equal(m["holder_offsets"], img["holder_offsets"])
        assert np.array_equal(m["holders"], img["holders"])
        assert all(np.array_equal(x, y) for a, b in zip(m["class_lists"], wire.class_lists(img))
                   for x, y in zip(a, b))


def test_merge_holder_counts_kernel(cp, ref):
    """The sharded plan's holder-offset merge (clairplan_merge_holder_counts) against its
    definition: global offsets = exclusive scan of the per-sample totals, rank r's starts =
    offsets + the counts of ranks < r."""
    import ctypes as C
    import torch
    L = cp.lib()
    L.clairplan_merge_holder_counts.argtypes = [C.c_void_p, C.c_void_p, C.c_uint32, C.c_uint32,
                                                C.c_void_p, C.c_void_p, C.c_void_p]
    rng = np.random.default_rng(4)
    for F, world in ((40_000, 4), (1_281_167, 8), (5, 3), (262_144, 2)):
        sizes = ref.generate_sizes(F, 0.1, 0.1, None, 1)
        p = cp.Plan(1, F, cp.PartitionSpec(2, 2, 1, True), [1.0], sizes)
        allc = rng.integers(0, 90, (world, F)).astype(np.int32)
        d_allc = torch.from_numpy(allc).cuda()
        tot = allc.astype(np.int64).sum(axis=0)
        want_glob = np.concatenate([[0], np.cumsum(tot)])
        for r in range(world):
            glob = torch.empty(F + 1, dtype=torch.int64, device="cuda")
            starts = torch.empty(F, dtype=torch.int64, device="cuda")
            cp._check(L.clairplan_merge_holder_counts(p._h, C.c_void_p(d_allc.data_ptr()), world, r,
                                                      C.c_void_p(glob.data_ptr()),
                                                      C.c_void_p(starts.data_ptr()), None))
            torch.cuda.synchronize()
            p_ = p  # the handle's stream was used: wait for it through a library sync
            assert np.array_equal(glob.cpu().numpy(), want_glob), (F, world, r)
            assert np.array_equal(starts.cpu().numpy(), want_glob[:-1] + allc[:r].astype(np.int64).sum(axis=0)), (F, r)
        p.close()


def test_rejection_kat_device(cp):
    """Epochs whose shuffle hits a Lemire rejection (found with tools/find_rejection, digests
    from the reference): the device path resolves them bit-exactly."""
    import hashlib
    import json
    with open(os.path.join(HERE, "golden", "rejection_kat.json")) as f:
        kat = json.load(f)
    for e in kat["epochs"]:
        p = cp.epoch_permutation(kat["seed"], e["epoch"], kat["samples"])
        assert hashlib.sha256(p.tobytes()).hexdigest() == e["sha256"], e["epoch"]


def test_build_from_perms_matches_build(cp, ref):
    """The sharded path on one GPU: permutation rows generated in two epoch ranges, then the
    worker-range build from those rows == the plain build of the same worker range."""
    import ctypes as C
    import torch
    F, N, B, E = 5000, 12, 120, 9
    sizes = ref.generate_sizes(F, 0.1, 0.1, None, 1)
    part = cp.PartitionSpec(N, B, E, True)
    L = cp.lib()
    L.clairplan_generate_perms.argtypes = [C.c_void_p, C.c_uint32, C.c_uint32, C.c_void_p]
    L.clairplan_build_from_perms.argtypes = [C.c_void_p, C.c_void_p]
    L.clairplan_holder_counts.argtypes = [C.c_void_p, C.c_void_p]
    for wr in ((0, 12), (3, 8)):
        a = cp.Plan(7, F, part, [8.0, 30.0], sizes, worker_range=wr).build()
        b = cp.Plan(7, F, part, [8.0, 30.0], sizes, worker_range=wr)
        rows = torch.empty((E, F), dtype=torch.int32, device="cuda")
        cp._check(L.clairplan_generate_perms(b._h, 0, 4, C.c_void_p(rows.data_ptr())))
        cp._check(L.clairplan_generate_perms(b._h, 4, E - 4, C.c_void_p(rows[4].data_ptr())))
        torch.cuda.synchronize()
        for e in (0, 5, 8):
            assert np.array_equal(rows[e].cpu().numpy().astype(np.uint32), ref.epoch_permutation(7, e, F))
        cp._check(L.clairplan_build_from_perms(b._h, C.c_void_p(rows.data_ptr())))
        assert np.array_equal(a.streams_flat(), b.streams_flat())
        for x, y in zip(a.class_lists(), b.class_lists()):
            assert all(np.array_equal(u, v) for u, v in zip(x, y))
        ha, hb = a.holders(), b.holders()
        assert np.array_equal(ha[0], hb[0]) and np.array_equal(ha[1], hb[1])
        cnt = torch.empty(F, dtype=torch.int32, device="cuda")
        cp._check(L.clairplan_holder_counts(b._h, C.c_void_p(cnt.data_ptr())))
        assert np.array_equal(np.diff(ha[0].astype(np.int64)), cnt.cpu().numpy())
        a.close()
        b.close()


def test_config4_imagenet22k_full_plan_against_reference(cp, ref):
    """Config 4 (ImageNet-22k shape, 90 epochs, 1024 workers; the north-star shape) in full:
    every stream, every worker's class lists (prefetch orders) and the whole holder CSR equal
    the reference's own per-worker plan (epoch_permutation, access_frequencies,
    nopfs_assign_caches per worker on all host threads, then the reference's build_index;
    policies.cpp:144-166, checked equal to the verbatim composition in test_oracle.py)."""
    F, N, b, E = 14_197_122, 1024, 32, 90
    caps = [120_000.0, 900_000.0]
    sizes = ref.generate_sizes(F, 0.1077, 0.2, 1_500_000.0, 1)
    p = cp.Plan(42, F, cp.PartitionSpec(N, b * N, E, True), caps, sizes).build()
    st = p.stats()
    assert st["accesses"] == 1_276_968_960 and st["path"] == "tier"
    flat = p.streams_flat()
    cl = p.class_lists()
    offs, hold = p.holders()
    p.close()
    a = ref.plan(42, F, N, b * N, E, True, caps, sizes, mode=1, threads=os.cpu_count() or 8)
    o = 0
    for w in range(N):
        n = len(a.streams[w])
        assert np.array_equal(flat[o:o + n], a.streams[w]), w
        o += n
    assert o == len(flat)
    del flat
    for w in range(N):
        for j in range(2):
            assert np.array_equal(cl[w][j], a.class_lists[w][j]), (w, j)
    del cl
    assert st["pairs"] == int(sum(len(x) for lists in a.class_lists for x in lists))
    assert np.array_equal(offs.astype(np.uint64), a.holder_offsets.astype(np.uint64))
    assert np.array_equal(hold, a.holders)


def test_config5_worker_subset_against_reference(cp, ref):
    """Config 5 (100 M samples, 100 epochs, 8192 workers): a full plan needs the
    sharded build (2^32 or more accesses); here the worker ranges [0, 512) and [7680, 8192)
    are built on one GPU and 64 workers inside them (both ends and both range edges included)
    are compared with the reference's own functions: streams, class lists and the
    subset-restricted holder CSR (a subsequence of the full CSR: holders are worker-ordered).
    The reference side never holds the 100 permutations together (epoch by epoch)."""
    F, E, N, b, R = 100_000_000, 100, 8192, 32, 512
    caps = [120_000.0, 900_000.0]
    sizes = ref.generate_sizes(F, 0.1077, 0.1, None, 1)
    rng = np.random.default_rng(5)
    subset = {0, 1, 2, R - 1, N - R, N - R + 1, N - 2, N - 1}
    while len(subset) < 64:
        subset.add(int(rng.integers(0, R)) if len(subset) % 2 else int(rng.integers(N - R, N)))
    subset = np.array(sorted(subset), np.uint32)
    a = ref.plan_subset_lowmem(42, F, N, b * N, E, True, caps, sizes, subset, os.cpu_count() or 8)
    roffs = a.holder_offsets.astype(np.int64)
    rowner = np.repeat(np.arange(F, dtype=np.int64), np.diff(roffs))
    for wr in ((0, R), (N - R, N)):
        sub = subset[(subset >= wr[0]) & (subset < wr[1])]
        p = cp.Plan(42, F, cp.PartitionSpec(N, b * N, E, True), caps, sizes, worker_range=wr).build()
        for w in sub:
            assert np.array_equal(p.stream(int(w)), a.streams[w]), w
        cl = p.class_lists()
        for w in sub:
            for j in range(2):
                assert np.array_equal(cl[int(w) - wr[0]][j], a.class_lists[w][j]), (w, j)
        offs, hold = p.holders()
        p.close()
        keep = np.isin(hold[:, 0], sub)
        owner = np.repeat(np.arange(F, dtype=np.int64), np.diff(offs.astype(np.int64)))
        rkeep = np.isin(a.holders[:, 0], sub)
        assert np.array_equal(owner[keep], rowner[rkeep]), wr
        assert np.array_equal(hold[keep], a.holders[rkeep]), wr


def test_concurrent_handles_from_host_threads(cp, ref):
    """The sweep pool calls the planner from several host threads at once
    (simulator.cpp:471-480 -> policies.cpp:454): four threads build four different plans on
    their own handles concurrently (ctypes releases the GIL); each equals the reference."""
    import threading
    cases = [(42, 20_000, 8, 256, 12, True, [150.0, 400.0]),
             (7, 30_011, 12, 120, 9, False, [60.0, 900.0]),
             (11, 25_000, 16, 512, 7, True, [1e6, 1e6]),
             (3, 40_000, 5, 100, 10, True, [20.0, 80.0, 300.0])]
    sizes = [ref.generate_sizes(c[1], 0.1077, 0.2, None, 1 + i) for i, c in enumerate(cases)]
    out = [None] * len(cases)
    errs = []

    def run(i):
        try:
            seed, F, N, B, E, dl, caps = cases[i]
            for _ in range(3):  # several builds per handle, interleaved with the other threads
                out[i] = device_plan(cp, seed, F, N, B, E, dl, caps, sizes[i])
        except Exception as ex:  # noqa: BLE001 - reported below
            errs.append((i, ex))

    ts = [threading.Thread(target=run, args=(i,)) for i in range(len(cases))]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errs, errs
    for i, (seed, F, N, B, E, dl, caps) in enumerate(cases):
        want = ref.plan(seed, F, N, B, E, dl, caps, sizes[i])
        assert plans_equal(want, out[i]) is None, i


def test_build_export_matches_separate_exports(cp, ref):
    """clairplan_build_export (sizes H2D + build + overlapped D2H) == build + the export calls."""
    import ctypes as C
    F, N, B, E = 30_000, 12, 240, 9
    sizes = ref.generate_sizes(F, 0.1077, 0.2, None, 1)
    # all-fit path; tier path with rejects left over; tier path whose last class takes every
    # reject (the class lists are then copied out during the build)
    for caps in ([1e6, 1e6], [20.0, 60.0], [100.0, 1e6]):
        p = cp.Plan(5, F, cp.PartitionSpec(N, B, E, True), caps, sizes).build()
        st = p.stats()
        want_streams = np.concatenate([p.stream(w) for w in range(N)])
        want_cl = np.concatenate([x for lists in p.class_lists() for x in lists])
        want_off, want_hold = p.holders()
        L = cp.lib()
        u32, u64 = C.POINTER(C.c_uint32), C.POINTER(C.c_uint64)
        L.clairplan_build_export.argtypes = [C.c_void_p, C.c_void_p, u32, C.c_uint64, u32,
                                             C.c_uint64, u64, u32, C.c_uint64]
        hs = np.zeros(st["accesses"], np.uint32)
        hc = np.zeros(max(st["holders"], 1), np.uint32)
        ho = np.zeros(F + 1, np.uint64)
        hh = np.zeros(3 * max(st["holders"], 1), np.uint32)
        hsz = np.ascontiguousarray(sizes, np.float64)
        cp._check(L.clairplan_build_export(p._h, hsz.ctypes.data_as(C.c_void_p),
                                           hs.ctypes.data_as(u32), len(hs), hc.ctypes.data_as(u32),
                                           len(hc), ho.ctypes.data_as(u64), hh.ctypes.data_as(u32),
                                           st["holders"]))
        assert np.array_equal(hs, want_streams)
        assert np.array_equal(hc[:len(want_cl)], want_cl)
        assert np.array_equal(ho, want_off.astype(np.uint64))
        assert np.array_equal(hh[:3 * st["holders"]], want_hold.reshape(-1))
        p.close()


@pytest.mark.parametrize("F,N,b,E,dl,caps", [
    (20_011, 9, 3, 7, False, None),
    (262_144, 64, 16, 10, True, None),
    (262_144, 64, 16, 10, True, [50.0, 1e9]),   # tier path (capacity-limited first fit)
    (1_281_167, 256, 32, 9, True, None),
    (65_536, 4096, 1, 3, True, None),           # 2048-worker shard: 64 bitmap words per sample
])
@pytest.mark.parametrize("dense", ["0", "1"])
def test_sharded_build_from_streams(cp, ref, monkeypatch, F, N, b, E, dl, caps, dense):
    """One rank's share of the multi-GPU build on one GPU: a worker-range
    handle fed its workers' streams of every epoch (what the all-to-all delivers, one source)
    through clairplan_generate_streams / clairplan_build_from_streams, with the sparse (CSR)
    or dense sample-major passes forced.  Its streams, class lists and holder records must
    equal the full single-GPU plan's restricted to those workers (the full plan is checked
    against the reference by the tests above)."""
    import ctypes as C
    import torch
    monkeypatch.setenv("CLAIRPLAN_DENSE", dense)
    sizes = cp.generate_sizes(F, 0.1077, 0.1, None, 1)
    part = cp.PartitionSpec(N, b * N, E, dl)
    caps = caps or [120.0 * F / 1e4, 900.0 * F / 1e4]
    full = cp.Plan(42, F, part, caps, sizes).build()
    st_full = full.streams_flat()
    offs_full, hold_full = full.holders()
    cl_full = full.class_lists()
    # the full plan the shards are compared with is itself the reference's (policies.cpp:144-166)
    want = ref.plan(42, F, N, b * N, E, dl, caps, sizes, mode=1, threads=os.cpu_count() or 8)
    assert np.array_equal(st_full, np.concatenate(want.streams))
    assert all(np.array_equal(x, y) for a, c in zip(want.class_lists, cl_full) for x, y in zip(a, c))
    assert np.array_equal(offs_full.astype(np.uint64), want.holder_offsets.astype(np.uint64))
    assert np.array_equal(hold_full, want.holders)
    samp = np.repeat(np.arange(F), np.diff(offs_full.astype(np.int64)))
    L = cp.lib()
    L.clairplan_generate_streams.argtypes = [C.c_void_p, C.c_uint32, C.c_uint32, C.c_void_p]
    L.clairplan_build_from_streams.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint32]
    L.clairplan_epoch_prefix.argtypes = [C.c_void_p, C.c_uint32, C.POINTER(C.c_uint64)]
    for wb, we in [(0, N // 2), (N // 2, N), (N // 3, N // 3 + max(1, N // 5))]:
        sh = cp.Plan(42, F, part, caps, sizes, worker_range=(wb, we))
        allst = torch.empty(len(st_full), dtype=torch.int32, device="cuda")
        cp._check(L.clairplan_generate_streams(sh._h, 0, E, C.c_void_p(allst.data_ptr())))
        pre = []
        for w in (wb, we):
            v = C.c_uint64()
            cp._check(L.clairplan_epoch_prefix(sh._h, w, C.byref(v)))
            pre.append(int(v.value))
        recv = allst[pre[0] * E:pre[1] * E]
        bounds = np.array([0, E], np.uint32)
        cp._check(L.clairplan_build_from_streams(sh._h, C.c_void_p(recv.data_ptr()),
                                                 bounds.ctypes.data_as(C.c_void_p), 1))
        torch.cuda.synchronize()
        lo = L.clairplan_stream_offset(full._h, wb)
        hi = L.clairplan_stream_offset(full._h, we)
        assert np.array_equal(sh.streams_flat(), st_full[lo:hi]), (wb, we)
        cl = sh.class_lists()
        assert all(np.array_equal(x, y) for a, c in zip(cl_full[wb:we], cl) for x, y in zip(a, c))
        offs, hold = sh.holders()
        m = (hold_full[:, 0] >= wb) & (hold_full[:, 0] < we)
        assert np.array_equal(hold, hold_full[m]), (wb, we)
        assert np.array_equal(np.diff(offs.astype(np.int64)), np.bincount(samp[m], minlength=F))
        sh.close()
        del allst
    full.close()
