"""Regenerates the golden vectors of tests/golden/ from the reference itself.

Run in the build container (needs /root/reference to compile oracle/_ref):
    python tests/golden/make_golden.py
The three permutation fixtures reproduce the reference's own
proj/tests/fixtures/perm_seed42_*.txt (checked by tests/test_oracle.py when the reference
tree is present) and the RNG values are the ones frozen in proj/tests/test_rng.cpp:12-22.
"""
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from _oracle import PERM_TAG, Ref  # noqa: E402


def main():
    r = Ref()
    for seed, epoch, F in ((42, 0, 8), (42, 1, 8), (42, 0, 16)):
        p = r.epoch_permutation(seed, epoch, F)
        with open(os.path.join(HERE, f"perm_seed{seed}_epoch{epoch}_f{F}.txt"), "w") as f:
            f.write(" ".join(str(int(x)) for x in p) + "\n")
    rng = {
        "seed42_perm_pos0": [hex(int(x)) for x in r.rng_stream(42, PERM_TAG, 0, 4)],
        "seed42_perm_epoch1": [hex(int(x)) for x in r.rng_stream(42, PERM_TAG, 1 << 34, 2)],
    }
    with open(os.path.join(HERE, "rng_kat.json"), "w") as f:
        json.dump(rng, f, indent=1)
    # Lemire-rejection KAT (rng.hpp:54-60): epochs found by tools/find_rejection on a B200
    # (F = 16,777,259, seed 42); the permutation digests come from the reference itself.
    import hashlib
    F, seed = 16_777_259, 42
    kat = {"samples": F, "seed": seed, "epochs": []}
    for epoch, step in ((66486, 11002896), (108120, 8809816), (118368, 4995318)):
        p = r.epoch_permutation(seed, epoch, F)
        kat["epochs"].append({"epoch": epoch, "rejecting_step": step,
                              "sha256": hashlib.sha256(p.tobytes()).hexdigest(),
                              "head": [int(x) for x in p[:8]]})
    with open(os.path.join(HERE, "rejection_kat.json"), "w") as f:
        json.dump(kat, f, indent=1)
    print("golden vectors written to", HERE)


if __name__ == "__main__":
    main()
