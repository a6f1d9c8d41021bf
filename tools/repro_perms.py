"""Single-GPU repro of one rank's perms-mode shuffle (clairplan_generate_perms on a
worker-range handle) for a given epoch range."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2101_08734_b200 import clairplan as cp  # noqa: E402

e0, n = int(sys.argv[1]), int(sys.argv[2])
wr = (int(sys.argv[3]), int(sys.argv[4]))
F, N, b, E = (int(x) for x in sys.argv[5:9]) if len(sys.argv) > 8 else (1_281_167, 256, 32, 9)
sizes = cp.generate_sizes(F, 0.1077, 0.1, None, 1)
p = cp.Plan(42, F, cp.PartitionSpec(N, b * N, E, True), [120.0 * F / 1e4, 900.0 * F / 1e4], sizes,
            worker_range=wr)
L = cp.lib()
L.clairplan_generate_perms.argtypes = [C.c_void_p, C.c_uint32, C.c_uint32, C.c_void_p]
rows = torch.empty((max(n, 1), F), dtype=torch.int32, device="cuda")
cp._check(L.clairplan_generate_perms(p._h, e0, n, C.c_void_p(rows.data_ptr())))
torch.cuda.synchronize()
for k in range(n):
    assert np.array_equal(rows[k].cpu().numpy().astype(np.uint32), cp.epoch_permutation(42, e0 + k, F))
print("perms ok", e0, n, wr)
