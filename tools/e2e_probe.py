"""Where the end-to-end time of one config-4 plan goes: build_export vs build + each export
timed on its own (pinned host buffers, as bench.py's e2e leg).  python tools/e2e_probe.py [config]"""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2101_08734_b200 import clairplan as cp  # noqa: E402


def main():
    c = int(sys.argv[1]) if len(sys.argv) > 1 else 4
    cfg = bench.CONFIGS[c]
    mu, sd, tot = cfg["sizes"]
    sizes = cp.generate_sizes(cfg["F"], mu, sd, tot, 1)
    N = cfg["N"]
    part = cp.PartitionSpec(N, cfg["b"] * N, cfg["E"], True)
    plan = cp.Plan(bench.SEED, cfg["F"], part, list(bench.CAPS), sizes, device=0).build()
    st = plan.stats()
    F = cfg["F"]
    L = cp.lib()
    u32 = C.POINTER(C.c_uint32)
    u64 = C.POINTER(C.c_uint64)
    h_sizes = torch.from_numpy(np.ascontiguousarray(sizes)).pin_memory()
    h_stream = torch.empty(st["accesses"], dtype=torch.int32).pin_memory()
    h_cls = torch.empty(max(st["holders"], 1), dtype=torch.int32).pin_memory()
    h_off = torch.empty(F + 1, dtype=torch.int64).pin_memory()
    h_hold = torch.empty(max(st["holders"], 1) * 3, dtype=torch.int32).pin_memory()
    L.clairplan_build_export.argtypes = [C.c_void_p, C.c_void_p, u32, C.c_uint64, u32, C.c_uint64, u64, u32,
                                         C.c_uint64]

    def t(f, n=3):
        f()
        torch.cuda.synchronize()
        a = time.perf_counter()
        for _ in range(n):
            f()
        torch.cuda.synchronize()
        return (time.perf_counter() - a) / n * 1e3

    def bx():
        cp._check(L.clairplan_build_export(plan._h, C.c_void_p(h_sizes.data_ptr()),
                                           C.cast(h_stream.data_ptr(), u32), st["accesses"],
                                           C.cast(h_cls.data_ptr(), u32), st["holders"],
                                           C.cast(h_off.data_ptr(), u64), C.cast(h_hold.data_ptr(), u32),
                                           st["holders"]))
    print("build_export ms", round(t(bx), 1))
    print("build ms", round(t(lambda: cp._check(L.clairplan_build(plan._h))), 1))
    print("export_streams ms", round(t(lambda: cp._check(L.clairplan_export_streams(
        plan._h, C.cast(h_stream.data_ptr(), u32), st["accesses"]))), 1), "GB", st["accesses"] * 4 / 1e9)
    print("export_class_lists ms", round(t(lambda: cp._check(L.clairplan_export_class_lists(
        plan._h, C.cast(h_cls.data_ptr(), u32), st["holders"]))), 1), "GB", st["holders"] * 4 / 1e9)
    print("export_holders ms", round(t(lambda: cp._check(L.clairplan_export_holders(
        plan._h, C.cast(h_off.data_ptr(), u64), C.cast(h_hold.data_ptr(), u32), st["holders"]))), 1),
        "GB", st["holders"] * 12 / 1e9 + (F + 1) * 8 / 1e9)
    d = torch.empty(st["holders"] * 12, dtype=torch.uint8, device="cuda")
    hb = h_hold.view(torch.uint8)
    print("raw D2H of the holder bytes ms", round(t(lambda: hb.copy_(d, non_blocking=True)), 1))


if __name__ == "__main__":
    main()
