"""CPU suite: the oracle pinned to the reference's golden vectors and to the reference itself.

* ``Port`` = oracle/clairplan_oracle.c (plain-C restatement)
* ``Ref``  = the unmodified reference sources compiled into oracle/_ref/
"""
import json
import os

import numpy as np
import pytest

from _oracle import PERM_TAG, plans_equal

HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN = os.path.join(HERE, "golden")
REF_FIXTURES = "/root/reference/proj/tests/fixtures"

# proj/tests/test_rng.cpp:12-22 ("frozen from an independent Python implementation")
RNG_KAT = [0xAC8ECAE6BC73963F, 0x288BF821559FDC26, 0xEE4A3A7284D5094E, 0x3C2594A435FAACF4]
RNG_KAT_EPOCH1 = [0x48711DE4E8779D75, 0x15028E39A3D624FF]


def load_perm(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return np.array([int(x) for x in f.read().split()], np.uint32)


def py_stream(seed, tag, start, n):
    """Pure-Python restatement of rng.hpp:16-47 for the KAT."""
    M = (1 << 64) - 1

    def mix(z):
        z ^= z >> 30
        z = (z * 0xBF58476D1CE4E5B9) & M
        z ^= z >> 27
        z = (z * 0x94D049BB133111EB) & M
        return z ^ (z >> 31)

    key = mix(seed ^ mix(tag))
    return [mix((key + (start + i + 1) * 0x9E3779B97F4A7C15) & M) for i in range(n)]


def test_rng_kat_python_restatement():
    assert py_stream(42, PERM_TAG, 0, 4) == RNG_KAT
    assert py_stream(42, PERM_TAG, 1 << 34, 2) == RNG_KAT_EPOCH1


def test_rng_kat_reference(ref):
    assert [int(x) for x in ref.rng_stream(42, PERM_TAG, 0, 4)] == RNG_KAT
    assert [int(x) for x in ref.rng_stream(42, PERM_TAG, 1 << 34, 2)] == RNG_KAT_EPOCH1
    with open(os.path.join(GOLDEN, "rng_kat.json")) as f:
        g = json.load(f)
    assert [int(x, 16) for x in g["seed42_perm_pos0"]] == RNG_KAT


@pytest.mark.parametrize("name,seed,epoch,F", [
    ("perm_seed42_epoch0_f8.txt", 42, 0, 8),
    ("perm_seed42_epoch1_f8.txt", 42, 1, 8),
    ("perm_seed42_epoch0_f16.txt", 42, 0, 16),
])
def test_perm_golden(port, ref, name, seed, epoch, F):
    g = load_perm(name)
    assert np.array_equal(port.epoch_permutation(seed, epoch, F), g)
    assert np.array_equal(ref.epoch_permutation(seed, epoch, F), g)
    if os.path.isdir(REF_FIXTURES):  # the committed fixture is the reference's own
        with open(os.path.join(REF_FIXTURES, name)) as f:
            assert np.array_equal(np.array(f.read().split(), np.uint32), g)


def test_perm_port_matches_reference(port, ref):
    rng = np.random.default_rng(1)
    for _ in range(300):
        F = int(rng.integers(1, 3000))
        seed = int(rng.integers(0, 2**63))
        e = int(rng.integers(0, 200))
        assert np.array_equal(port.epoch_permutation(seed, e, F), ref.epoch_permutation(seed, e, F))
    # test_access.cpp:27-37: single element / permutation property
    assert list(port.epoch_permutation(123, 0, 1)) == [0]
    assert sorted(port.epoch_permutation(5, 3, 10)) == list(range(10))


def test_sizes_port_matches_reference(port, ref):
    for args in [(5000, 0.1077, 0.1, 135000.0 * 5000 / 1281167, 1),
                 (3000, 0.1077, 0.2, 1e4, 7), (1000, 16.0, 0.0, None, 1),
                 (2000, 1.0, 0.4, None, 3)]:
        a = port.generate_sizes(*args)
        b = ref.generate_sizes(*args)
        assert np.array_equal(a.view(np.uint64), b.view(np.uint64))


CASES = [
    # seed, F, N, B, E, drop_last, caps, (mean, sigma)
    (42, 2000, 4, 128, 10, True, [20.0, 900.0], (0.1077, 0.1)),
    (7, 1500, 3, 7, 5, False, [5.0, 30.0], (0.1, 0.3)),
    (9, 1000, 16, 16, 6, True, [1e6, 1e6], (1.0, 0.0)),
    (1, 777, 5, 13, 4, False, [3.0], (0.5, 0.5)),
    (3, 600, 2, 9, 3, True, [2.0, 3.0, 40.0], (0.2, 0.1)),
    (11, 500, 4, 4, 20, True, [], (0.1, 0.1)),
]


@pytest.mark.parametrize("case", CASES)
def test_port_plan_matches_reference(port, ref, case):
    seed, F, N, B, E, dl, caps, (mu, sd) = case
    sizes = ref.generate_sizes(F, mu, sd, None, 1)
    a = ref.plan(seed, F, N, B, E, dl, caps, sizes)
    b = port.plan(seed, F, N, B, E, dl, caps, sizes)
    assert plans_equal(a, b) is None


@pytest.mark.parametrize("case", CASES[:4])
def test_reference_per_worker_harness_matches_verbatim(ref, case):
    """The threaded per-worker harness (CPU baseline / large configs) == verbatim path."""
    seed, F, N, B, E, dl, caps, (mu, sd) = case
    sizes = ref.generate_sizes(F, mu, sd, None, 1)
    a = ref.plan(seed, F, N, B, E, dl, caps, sizes, mode=0)
    b = ref.plan(seed, F, N, B, E, dl, caps, sizes, mode=1, threads=4)
    assert plans_equal(a, b) is None


@pytest.mark.parametrize("case", CASES[:4])
def test_reference_lowmem_subset_harness(ref, case):
    """The epoch-by-epoch subset harness (config 5 checks) == the subset harness: subset
    streams, class lists and the subset-restricted holder CSR."""
    seed, F, N, B, E, dl, caps, (mu, sd) = case
    sizes = ref.generate_sizes(F, mu, sd, None, 1)
    subset = np.array(sorted({0, N - 1, N // 2}), np.uint32)
    a = ref.plan_subset(seed, F, N, B, E, dl, caps, sizes, subset, 4)
    b = ref.plan_subset_lowmem(seed, F, N, B, E, dl, caps, sizes, subset, 4)
    for w in subset:
        assert np.array_equal(a.streams[w], b.streams[w])
        for j in range(len(caps)):
            assert np.array_equal(a.class_lists[w][j], b.class_lists[w][j])
    assert np.array_equal(a.holder_offsets, b.holder_offsets)
    assert np.array_equal(a.holders, b.holders)


def test_port_generic_assign_matches_reference(port, ref):
    # test_policies.cpp:54-67: hand-built stream, counts {5, 2}, class 1 fits one sample
    streams = [np.array([0, 1, 0, 0, 1, 0, 0], np.uint32)]
    counts = np.array([[5, 2]], np.uint32)
    a = ref.assign_from_streams(streams, counts, [1.0, 10.0], [1.0, 1.0])
    b = port.assign_from_streams(streams, counts, [1.0, 10.0], [1.0, 1.0])
    assert list(a.class_lists[0][0]) == [0] and list(a.class_lists[0][1]) == [1]
    assert plans_equal(a, b, check_streams=False) is None
    # inconsistent tables: counts > 0 for samples absent from the stream, ties by index
    rng = np.random.default_rng(5)
    for _ in range(20):
        N, F = int(rng.integers(1, 5)), int(rng.integers(5, 60))
        streams = [rng.integers(0, F, int(rng.integers(0, 80))).astype(np.uint32) for _ in range(N)]
        counts = rng.integers(0, 4, (N, F)).astype(np.uint32)
        sizes = rng.uniform(0.1, 2.0, F)
        caps = [float(rng.uniform(1, 10)), float(rng.uniform(1, 30))]
        a = ref.assign_from_streams(streams, counts, caps, sizes)
        b = port.assign_from_streams(streams, counts, caps, sizes)
        assert plans_equal(a, b, check_streams=False) is None


def _kat():
    with open(os.path.join(GOLDEN, "rejection_kat.json")) as f:
        return json.load(f)


def test_rejection_kat_oracle(port):
    """Lemire rejection (rng.hpp:54-60) KAT: the C restatement reproduces the reference's
    permutation digest, and ignoring the rejection would change it."""
    import hashlib
    kat = _kat()
    e = kat["epochs"][0]
    p = port.epoch_permutation(kat["seed"], e["epoch"], kat["samples"])
    assert hashlib.sha256(p.tobytes()).hexdigest() == e["sha256"]
    assert [int(x) for x in p[:8]] == e["head"]
    naive = port.epoch_permutation_norej(kat["seed"], e["epoch"], kat["samples"])
    assert hashlib.sha256(naive.tobytes()).hexdigest() != e["sha256"]
