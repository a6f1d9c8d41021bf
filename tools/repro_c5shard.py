"""One rank's share of config 5 at 4 ranks (workers [0, 2048): 2.5e9 local entries) built on
one GPU through clairplan_generate_streams + clairplan_build_from_streams."""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2101_08734_b200 import clairplan as cp  # noqa: E402

F, N, b, E = 100_000_000, 8192, 32, 100
nw = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
sizes = cp.generate_sizes(F, 0.1077, 0.1, None, 1)
part = cp.PartitionSpec(N, b * N, E, True)
L = cp.lib()
L.clairplan_generate_streams.argtypes = [C.c_void_p, C.c_uint32, C.c_uint32, C.c_void_p]
L.clairplan_build_from_streams.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint32]
L.clairplan_epoch_prefix.argtypes = [C.c_void_p, C.c_uint32, C.POINTER(C.c_uint64)]
sh = cp.Plan(42, F, part, [120_000.0, 900_000.0], sizes, worker_range=(0, nw))
v = C.c_uint64()
cp._check(L.clairplan_epoch_prefix(sh._h, nw, C.byref(v)))
loc = int(v.value) * E
recv = torch.empty(loc, dtype=torch.int32, device="cuda")
# the rank's own workers' entries of every epoch, epoch by epoch through a per-epoch buffer
allst = torch.empty(int(v.value) * 0 + (F // (b * N)) * b * N, dtype=torch.int32, device="cuda")
t = time.time()
pre_all = C.c_uint64()
cp._check(L.clairplan_epoch_prefix(sh._h, N, C.byref(pre_all)))
per_epoch_all = int(pre_all.value)
for e in range(E):
    cp._check(L.clairplan_generate_streams(sh._h, e, 1, C.c_void_p(allst.data_ptr())))
    torch.cuda.synchronize()
    recv[e * int(v.value):(e + 1) * int(v.value)] = allst[:int(v.value)]
torch.cuda.synchronize()
print("streams generated", round(time.time() - t, 1), "s; local entries", loc, flush=True)
bounds = np.array([0, E], np.uint32)
try:
    cp._check(L.clairplan_build_from_streams(sh._h, C.c_void_p(recv.data_ptr()),
                                             bounds.ctypes.data_as(C.c_void_p), 1))
    st = sh.stats()
    print("built", st, flush=True)
except Exception as ex:
    print("build failed:", ex, flush=True)
# sample-side view of the received streams: every entry a valid sample id?
mx = int(recv.max().item()) if recv.numel() else 0
mn = int(recv.min().item()) if recv.numel() else 0
print("recv min/max", mn, mx, "F", F, flush=True)
