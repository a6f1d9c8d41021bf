"""B200-native NoPFS clairvoyant plan build (arXiv 2101.08734) — see DESIGN.md.

The product is ``libclairplan.so`` (hand-written sm_100a CUDA behind the C ABI in
``include/clairplan.h``); ``clairplan`` is the Python mirror of the reference's clairsim API.
"""
from .clairplan import (  # noqa: F401
    AccessStream,
    CacheAssignment,
    FrequencyTable,
    PartitionSpec,
    Plan,
    REFERENCE_CAPACITIES_MB,
    access_frequencies,
    all_access_counts,
    batch_slice,
    build_access_streams,
    epoch_permutation,
    generate_sizes,
    nopfs_assign_caches,
    validate,
    worker_access_counts,
)
