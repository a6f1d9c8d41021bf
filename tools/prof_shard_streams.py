"""One rank's share of the sharded (streams) build emulated on one GPU: a handle for the first
1/G of the workers is fed all epochs' streams of its workers (what the all-to-all delivers)
and built `reps` times.  Prints the stage times; run under ncu for a launch list.
    python tools/prof_shard_streams.py [config] [reps] [G]     (CLAIRPLAN_DENSE=1: dense passes)"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2101_08734_b200 import clairplan as cp  # noqa: E402


def main():
    c = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    G = int(sys.argv[3]) if len(sys.argv) > 3 else 8
    cfg = bench.CONFIGS[c]
    mu, sd, tot = cfg["sizes"]
    sizes = cp.generate_sizes(cfg["F"], mu, sd, tot, 1)
    N, E = cfg["N"], cfg["E"]
    part = cp.PartitionSpec(N, cfg["b"] * N, E, True)
    plan = cp.Plan(bench.SEED, cfg["F"], part, list(bench.CAPS), sizes, device=0,
                   worker_range=(0, N // G))
    L = cp.lib()
    L.clairplan_generate_streams.argtypes = [C.c_void_p, C.c_uint32, C.c_uint32, C.c_void_p]
    L.clairplan_build_from_streams.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint32]
    allst = torch.empty(bench.accesses_of(cfg), dtype=torch.int32, device="cuda")
    cp._check(L.clairplan_generate_streams(plan._h, 0, E, C.c_void_p(allst.data_ptr())))
    bounds = np.array([0, E], np.uint32)
    for _ in range(reps):
        cp._check(L.clairplan_build_from_streams(plan._h, C.c_void_p(allst.data_ptr()),
                                                 bounds.ctypes.data_as(C.c_void_p), 1))
    torch.cuda.synchronize()
    L.clairplan_stage_times.argtypes = [C.c_void_p, C.POINTER(C.c_double), C.c_uint32]
    L.clairplan_stage_name.restype = C.c_char_p
    buf = (C.c_double * 16)()
    ns = L.clairplan_stage_times(plan._h, buf, 16)
    st = plan.stats()
    print("G", G, "device_ms", round(st["device_ms"], 3), st["path"],
          {L.clairplan_stage_name(i).decode(): round(buf[i], 3) for i in range(ns)})


if __name__ == "__main__":
    main()
