import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2101_08734_b200 import clairplan as cp  # noqa: E402

F, N, b, E = 20000, 7, 5, 13
scen = sys.argv[1]
L = cp.lib()
L.clairplan_generate_perms.argtypes = [C.c_void_p, C.c_uint32, C.c_uint32, C.c_void_p]
sizes = cp.generate_sizes(F, 0.1077, 0.1, None, 1)
p = cp.Plan(42, F, cp.PartitionSpec(N, b * N, E, True), [12.0, 90.0], sizes, worker_range=(5, 7))
e0, n = (10, 3) if scen != "b" else (0, 4)
rows = torch.zeros((4, F), dtype=torch.int32, device="cuda")
if scen in ("a", "b", "c"):
    cp._check(L.clairplan_generate_perms(p._h, e0, n, C.c_void_p(rows.data_ptr())))
    torch.cuda.synchronize()
    print(scen, "generate ok", flush=True)
    r = rows.cpu().numpy().astype(np.uint32)
    print(scen, "row sorted ok", [bool(np.array_equal(np.sort(r[k]), np.arange(F))) for k in range(n)], flush=True)
if scen == "c":
    p.close()
for k in range(n):
    try:
        x = cp.epoch_permutation(42, e0 + k, F)
        print(scen, "epoch_permutation", e0 + k, "ok", bool(np.array_equal(x, rows[k].cpu().numpy().astype(np.uint32))), flush=True)
    except Exception as ex:
        print(scen, "epoch_permutation", e0 + k, "FAIL", ex, flush=True)
        break
