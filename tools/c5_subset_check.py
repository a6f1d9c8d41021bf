"""Config 5 (100 M samples, 100 epochs, 8192 workers) on one B200: handles for
the worker ranges [0, 512) and [7680, 8192) (a full plan of all 8192 workers needs the
8-GPU sharded build), checked bit-exactly against the reference's own functions for a worker
subset inside them: streams, class lists (prefetch orders) and the subset-restricted holder
CSR.  The reference side never holds the 100 permutations together (epoch by epoch).
    python tools/c5_subset_check.py [F] [E] [N] [range]"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from paper_2101_08734_b200 import clairplan as cp  # noqa: E402


def check_range(ref, F, E, N, wr, sizes, caps, subset):
    b = 32
    t0 = time.time()
    p = cp.Plan(42, F, cp.PartitionSpec(N, b * N, E, True), caps, sizes, worker_range=wr).build()
    st = p.stats()
    t1 = time.time()
    ok = True
    sub = [w for w in subset if wr[0] <= w < wr[1]]
    for w in sub:
        ok &= bool(np.array_equal(p.stream(w), ref.streams[w]))
    cl = p.class_lists()
    for w in sub:
        for j in range(len(caps)):
            ok &= bool(np.array_equal(cl[w - wr[0]][j], ref.class_lists[w][j]))
    offs, hold = p.holders()
    p.close()
    keep = np.isin(hold[:, 0], np.array(sub, np.uint32))
    owner = np.repeat(np.arange(F, dtype=np.int64), np.diff(offs.astype(np.int64)))
    mine_k, mine_h = owner[keep], hold[keep]
    roffs = ref.holder_offsets.astype(np.int64)
    rowner = np.repeat(np.arange(F, dtype=np.int64), np.diff(roffs))
    rkeep = np.isin(ref.holders[:, 0], np.array(sub, np.uint32))
    ok &= bool(np.array_equal(rowner[rkeep], mine_k) and np.array_equal(ref.holders[rkeep], mine_h))
    print(f"range {wr}: device build {st['device_ms']:.1f} ms (wall {t1 - t0:.1f} s), A {st['accesses']}, "
          f"D {st['pairs']}, path {st['path']}, subset {len(sub)} workers, holders {keep.sum()}, "
          f"ok={ok}", flush=True)
    return ok


def main():
    F = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000_000
    E = int(sys.argv[2]) if len(sys.argv) > 2 else 100
    N = int(sys.argv[3]) if len(sys.argv) > 3 else 8192
    R = int(sys.argv[4]) if len(sys.argv) > 4 else 512
    caps = [120_000.0, 900_000.0]
    sizes = cp.generate_sizes(F, 0.1077, 0.1, None, 1)
    rng = np.random.default_rng(5)
    ranges = [(0, R), (N - R, N)]
    subset = sorted(set([0, 1, 2, R - 1, N - R, N - R + 1, N - 2, N - 1] +
                        [int(x) for x in rng.integers(0, R, 10)] +
                        [int(x) for x in rng.integers(N - R, N, 10)]))
    from _oracle import Ref
    t0 = time.time()
    ref = Ref().plan_subset_lowmem(42, F, N, 32 * N, E, True, caps, sizes,
                                   np.array(subset, np.uint32), os.cpu_count() or 8)
    print(f"reference subset ({len(subset)} workers) {time.time() - t0:.1f} s", flush=True)
    ok = all(check_range(ref, F, E, N, wr, sizes, caps, subset) for wr in ranges)
    print("c5_subset_check", "OK" if ok else "FAILED", "F", F, "E", E, "N", N)
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
