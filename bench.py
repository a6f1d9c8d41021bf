#!/usr/bin/env python
"""Benchmark of the NoPFS clairvoyant plan build (BASELINE.json metric).

A step = one full plan build (seed -> every epoch's permutation -> per-worker access
streams -> (count, first-access) per (worker, sample) -> tier assignment -> prefetch orders
-> holder CSR).  Default workload: the ImageNet-22k shape, 14,197,122 samples, 90 epochs,
1024 workers, per-worker batch 32 (BASELINE.json configs[3], the north-star shape and the
largest configuration that builds on one B200; `--config N` selects another).  `value` =
sample accesses per second of the device-resident build (sizes already in HBM), timed with
the library's CUDA events on its stream; `e2e` is the same plan through the C ABI with host
buffers (sizes H2D, every output D2H) inside the timed region.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config C]

Multi-GPU (torchrun, one rank per GPU, paper_2101_08734_b200/distributed.py): every rank
generates the streams of its epoch range, the stream slices move to the ranks owning their
workers over NVLink, every rank builds the plan of its contiguous worker range and the holder
CSR offsets are merged with an NCCL all-gather of the per-sample holder counts; time = max
over ranks (strong scaling: the same configuration at every N).

The reference arm (`--impl reference`) and the `cpu_baseline` leg run the reference's own
C++ functions (oracle/_ref) on all host threads over a bounded sample of the same workload
(see cpu_reference_sample).
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

CONFIGS = {
    # F, N, per-worker batch, E, sizes (mean, sigma, total)   -- BASELINE.md §5 / SURVEY §8(d)
    1: dict(F=1_281_167, N=4, b=32, E=10, sizes=(0.1077, 0.1, 135_000.0),
            name="imagenet1k-e10-n4"),
    2: dict(F=1_281_167, N=256, b=32, E=90, sizes=(0.1077, 0.1, 135_000.0),
            name="imagenet1k-e90-n256"),
    3: dict(F=262_144, N=1024, b=16, E=100, sizes=(16.0, 0.0, None), name="cosmoflow16-e100-n1024"),
    4: dict(F=14_197_122, N=1024, b=32, E=90, sizes=(0.1077, 0.2, 1_500_000.0),
            name="imagenet22k-e90-n1024"),
    5: dict(F=100_000_000, N=8192, b=32, E=100, sizes=(0.1077, 0.1, None),
            name="synthetic100m-e100-n8192"),
}
SEED = 42
CAPS = (120_000.0, 900_000.0)  # scenarios.cpp:25-40 (RAM, SSD); staging is class 0, unpacked
METRIC = "clairvoyant plan build: sample-accesses/sec and plan latency at 1/2/4/8 B200"
UNIT = "sample-accesses/s"


def dist_env():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("LOCAL_RANK", "0")),
            int(os.environ.get("WORLD_SIZE", "1")))


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def accesses_of(cfg):
    B = cfg["b"] * cfg["N"]
    return cfg["E"] * (cfg["F"] // B) * B


class ClockSampler:
    """SM clocks + throttle reasons sampled DURING the timed region (B200_PROFILING.md): NVML
    polled every ~2 ms from a thread (the timed region of a config-2 run is ~60-80 ms, shorter
    than nvidia-smi's sampling period); `nvidia-smi -lms 100` when NVML is unavailable."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.nvml = None
        self.lines = []
        self.samples = []  # NVML: (sm_mhz, reasons bitmask)
        self.stop_ev = threading.Event()

    def _nvml_handle(self):
        import pynvml
        pynvml.nvmlInit()
        try:
            uuid = str(torch.cuda.get_device_properties(self.gpu).uuid)
            return pynvml, pynvml.nvmlDeviceGetHandleByUUID(
                uuid if uuid.startswith("GPU-") else "GPU-" + uuid)
        except Exception:
            return pynvml, pynvml.nvmlDeviceGetHandleByIndex(self.gpu)

    def start(self):
        try:
            self.nvml, self.h = self._nvml_handle()
            N = self.nvml
            self.smax = float(N.nvmlDeviceGetMaxClockInfo(self.h, N.NVML_CLOCK_SM))
            self.bits = [N.nvmlClocksEventReasonHwSlowdown, N.nvmlClocksEventReasonHwThermalSlowdown,
                         N.nvmlClocksEventReasonSwThermalSlowdown, N.nvmlClocksEventReasonSwPowerCap]

            def poll():
                while not self.stop_ev.is_set():
                    try:
                        self.samples.append((float(N.nvmlDeviceGetClockInfo(self.h, N.NVML_CLOCK_SM)),
                                             int(N.nvmlDeviceGetCurrentClocksEventReasons(self.h))))
                    except Exception:
                        pass
                    time.sleep(0.002)

            self.t = threading.Thread(target=poll, daemon=True)
            self.t.start()
            return
        except Exception:
            self.nvml = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.nvml is not None:
            self.stop_ev.set()
            self.t.join(timeout=1)
            sm = [c for c, _ in self.samples]
            reasons = {n for _, r in self.samples for n, b in zip(self.NAMES, self.bits) if r & b}
            return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": self.smax,
                    "reasons": sorted(reasons), "samples": len(sm), "source": "nvml"}
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], None, set()
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax = float(parts[2])
            except ValueError:
                continue
            for n, v in zip(self.NAMES, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm), "source": "nvidia-smi"}


def cpu_reference_sample(cfg, sizes, threads):
    """The reference's own functions (oracle/_ref, per-worker harness on all host threads) on a
    bounded sample of the workload: every epoch's permutation and every worker's stream (the
    whole of those phases), then the assignment + build_index of an evenly spaced worker
    subset (all workers when N <= 2 * threads).  The assignment phase is linear in the
    workers, so the full-plan time is estimated as perms + streams + (assign + index) * N / S.
    Only this leg and --impl reference execute anything under oracle/."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from _oracle import Ref
    ref = Ref()
    N = cfg["N"]
    S = N if N <= 2 * threads else 2 * threads
    subset = np.unique(np.linspace(0, N - 1, S).round().astype(np.uint32))
    S = len(subset)
    t0 = time.perf_counter()
    ph = ref.time_subset(SEED, cfg["F"], N, cfg["b"] * N, cfg["E"], True, list(CAPS), sizes,
                         subset, threads)
    wall = time.perf_counter() - t0
    est = (ph[0] + ph[1] + (ph[2] + ph[3]) * N / S) / 1e3
    return {"est_s": est, "wall_s": wall, "subset": S, "phases_ms": [round(x, 1) for x in ph]}


def cpu_baseline_entry(cfg, smp, threads):
    A = accesses_of(cfg)
    exact = smp["subset"] == cfg["N"]
    how = ("full plan" if exact else
           f"{smp['subset']} of {cfg['N']} workers assigned, full-plan time = perms + streams + "
           f"(assign + build_index) x {cfg['N']}/{smp['subset']}")
    return {"value": A / smp["est_s"], "unit": UNIT, "cores": threads, "kind": "reference",
            "sample": f"{cfg['name']}: reference epoch_permutation for all {cfg['E']} epochs, "
                      f"every worker's stream, access_frequencies + nopfs_assign_caches + "
                      f"build_index per worker on {threads} host threads ({how}); "
                      f"phases ms {smp['phases_ms']}, sample wall {smp['wall_s']:.2f} s, "
                      f"estimated plan {smp['est_s']:.2f} s"}


def config_dict(cfg, world):
    """The `config` of both arms (identical for the same workload and N)."""
    return {"workload": cfg["name"], "samples": cfg["F"], "workers": cfg["N"],
            "per_worker_batch": cfg["b"], "epochs": cfg["E"], "seed": SEED,
            "capacities_mb": list(CAPS), "drop_last": True,
            "l2": "256 MB flush before every timed step (device arm)",
            "sharding": ("single GPU" if world == 1 else
                         f"epochs sharded over {world} GPUs for the permutations and stream "
                         "cutting, streams exchanged over NVLink, worker ranges for the rest, "
                         "holder offsets merged by NCCL all-gather")}


def run_reference(args, cfg):
    rank, _, world = dist_env()
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from _oracle import Ref  # sizes from the reference's own DatasetModel::generate
    mu, sd, tot = cfg["sizes"]
    sizes = Ref().generate_sizes(cfg["F"], mu, sd, tot, 1)
    for _ in range(args.warmup):
        cpu_reference_sample(cfg, sizes, threads)
    smps = [cpu_reference_sample(cfg, sizes, threads) for _ in range(args.steps)]
    smp = dict(smps[-1])
    smp["est_s"] = statistics.mean(x["est_s"] for x in smps)
    smp["wall_s"] = statistics.mean(x["wall_s"] for x in smps)
    cpu = cpu_baseline_entry(cfg, smp, threads)
    v = cpu["value"]
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": smp["est_s"] * 1e3,
        "sample_wall_ms_per_step": smp["wall_s"] * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u32",
        "data": "synthetic (seed-generated, BASELINE config shapes)",
        "config": config_dict(cfg, world),
        "cpu_baseline": cpu,
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))


def dominant_stage(stage_ms, A_loc, hbm):
    """The largest stage of the rank's last build (CUDA events on the library stream) against
    its compulsory bytes: the permutation stage writes the 4A stream bytes and nothing else is
    an input or output of the plan (the shuffle is seed-generated; its grouping arrays are
    implementation-internal)."""
    if not stage_ms:
        return None
    name = max(stage_ms, key=stage_ms.get)
    ms = stage_ms[name]
    alg = {"permutations+streams": 4.0 * A_loc}.get(name)
    if alg is None or ms <= 0:
        return {"name": name, "ms": ms}
    ach = alg / (ms * 1e-3) / 1e9
    return {"name": name, "ms": ms, "alg_bytes": alg, "achieved": ach, "unit": "GB/s",
            "frac": ach / hbm}


def run_ours(args, cfg):
    import torch
    from paper_2101_08734_b200 import clairplan as cp

    rank, local, world = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    N = cfg["N"]
    wb, we = rank * N // world, (rank + 1) * N // world
    mu, sd, tot = cfg["sizes"]
    sizes = cp.generate_sizes(cfg["F"], mu, sd, tot, 1)
    part = cp.PartitionSpec(N, cfg["b"] * N, cfg["E"], True)
    if world > 1:
        from paper_2101_08734_b200.distributed import DistributedPlan
        dplan = DistributedPlan(SEED, cfg["F"], part, list(CAPS), sizes,
                                mode=os.environ.get("CLAIRPLAN_DIST_MODE", "p2p"))
        plan = dplan.plan

        def build():
            dplan.build()

        def dplan_timings():  # host wall time of the last build's phases on this rank
            return dict(dplan.timings)
    else:
        plan = cp.Plan(SEED, cfg["F"], part, list(CAPS), sizes, device=local, worker_range=(wb, we))

        def build():
            plan.build()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")  # > 126 MB L2

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
            torch.cuda.synchronize()

    for _ in range(args.warmup):
        build()
    barrier()
    sampler = ClockSampler(local)
    sampler.start()
    dev_ms, stage = [], None
    launches = 0
    t_wall = time.perf_counter()
    for _ in range(args.steps):
        flush.fill_(1)
        torch.cuda.synchronize()
        if world > 1:
            # the sharded build spans the library stream and NCCL on torch's stream; every
            # library call synchronises its own stream, so events on torch's stream bracket it
            ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ev0.record()
            build()
            ev1.record()
            ev1.synchronize()
            dev_ms.append(ev0.elapsed_time(ev1))
        else:
            build()
            dev_ms.append(plan.stats()["device_ms"])
        st = plan.stats()
        launches += plan.launch_count()
    barrier()
    t_wall = time.perf_counter() - t_wall
    clocks = sampler.stop()
    stage_ms = {}
    import ctypes
    L = cp.lib()
    L.clairplan_stage_times.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_double),
                                        ctypes.c_uint32]
    L.clairplan_stage_name.restype = ctypes.c_char_p
    buf = (ctypes.c_double * 16)()
    ns = L.clairplan_stage_times(plan._h, buf, 16)
    for i in range(ns):
        stage_ms[L.clairplan_stage_name(i).decode()] = round(buf[i], 4)

    total_ms = float(sum(dev_ms))
    A_loc, D_loc = st["accesses"], st["pairs"]
    vec = torch.tensor([total_ms, float(A_loc), float(D_loc)], dtype=torch.float64, device="cuda")
    if world > 1:
        mx = vec.clone()
        torch.distributed.all_reduce(mx[:1], op=torch.distributed.ReduceOp.MAX)
        sm = vec.clone()
        torch.distributed.all_reduce(sm, op=torch.distributed.ReduceOp.SUM)
        total_ms, A_all, D_all = float(mx[0]), float(sm[1]), float(sm[2])
    else:
        A_all, D_all = float(A_loc), float(D_loc)
    ms_step = total_ms / args.steps
    value = A_all / (ms_step / 1e3)

    # ---- end to end through the C ABI with host buffers (rank-local)
    e2e = None
    if not args.no_e2e:
        e2e = e2e_measure(cp, plan, build, sizes, cfg, args, world, A_all)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        try:
            cpu = cpu_baseline_entry(cfg, cpu_reference_sample(cfg, sizes, threads), threads)
        except Exception as ex:  # no oracle/_ref on this box
            cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "reference",
                   "sample": f"unavailable: {ex}"}

    hbm, peak_kind = peaks()
    B_alg = 8 * A_all + 32 * D_all + 4 * (cfg["F"] + 1)
    achieved = B_alg / (ms_step / 1e3) / 1e9
    # DRAM bytes per plan of this workload from the committed ncu launch list of the same
    # build (an ncu capture cannot run inside the timed bench); null when none is committed
    traffic, traffic_src = None, None
    tpath = os.path.join(ROOT, "profiles", "traffic_latest.json")
    if os.path.exists(tpath) and world == 1:
        try:
            with open(tpath) as f:
                tw = json.load(f).get("workloads", {}).get(cfg["name"])
            if tw:
                traffic, traffic_src = tw["dram_bytes_per_plan"], tw["list"]
        except Exception:
            traffic = None
    if rank == 0:
        out = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "u32", "data": "synthetic (seed-generated, BASELINE config shapes)",
            "config": config_dict(cfg, world),
            "plan_latency_ms": ms_step,
            "wall_ms_per_step": t_wall * 1e3 / args.steps,
            "accesses": int(A_all), "pairs": int(D_all),
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm * world,
                         "unit": "GB/s", "frac": achieved / (hbm * world), "traffic": traffic,
                         "traffic_source": traffic_src,
                         "kernel": "whole plan pipeline (B_alg = 8A + 32D + 4(F+1) per plan)",
                         "peak_kind": f"{peak_kind} copy bandwidth x {world}",
                         "dominant_stage": dominant_stage(stage_ms, A_loc, hbm)},
            "stages_ms": stage_ms,
            "rank0_phases_ms": (dplan_timings() if world > 1 else None),
            "e2e": e2e,
            "cpu_baseline": cpu,
            "gpu_launches": launches,
            "clocks": clocks,
        }
        print(json.dumps(out))
    plan.close()
    if world > 1:
        torch.distributed.destroy_process_group()


def e2e_measure(cp, plan, build, sizes, cfg, args, world, A_all):
    """sizes H2D from pinned memory + build + every output D2H into pinned buffers."""
    import ctypes
    import torch
    L = cp.lib()
    L.clairplan_set_sizes.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]
    st = plan.stats()
    F = cfg["F"]
    h_sizes = torch.from_numpy(np.ascontiguousarray(sizes)).pin_memory()
    nloc = plan.wend - plan.wbegin
    h_stream = torch.empty(st["accesses"], dtype=torch.int32).pin_memory()
    h_cls = torch.empty(max(st["holders"], 1), dtype=torch.int32).pin_memory()
    h_off = torch.empty(F + 1, dtype=torch.int64).pin_memory()
    h_hold = torch.empty(max(st["holders"], 1) * 3, dtype=torch.int32).pin_memory()
    u32 = ctypes.POINTER(ctypes.c_uint32)
    u64 = ctypes.POINTER(ctypes.c_uint64)

    L.clairplan_build_export.argtypes = [ctypes.c_void_p, ctypes.c_void_p, u32, ctypes.c_uint64, u32,
                                         ctypes.c_uint64, u64, u32, ctypes.c_uint64]

    def step():
        if world == 1:  # one C-ABI call: sizes H2D, build, outputs D2H (stream copy overlapped)
            cp._check(L.clairplan_build_export(
                plan._h, ctypes.c_void_p(h_sizes.data_ptr()),
                ctypes.cast(h_stream.data_ptr(), u32), st["accesses"],
                ctypes.cast(h_cls.data_ptr(), u32), st["holders"],
                ctypes.cast(h_off.data_ptr(), u64), ctypes.cast(h_hold.data_ptr(), u32),
                st["holders"]))
            return
        cp._check(L.clairplan_set_sizes(plan._h, ctypes.c_void_p(h_sizes.data_ptr()), 0))
        build()
        cp._check(L.clairplan_export_streams(plan._h, ctypes.cast(h_stream.data_ptr(), u32),
                                             st["accesses"]))
        cp._check(L.clairplan_export_class_lists(plan._h, ctypes.cast(h_cls.data_ptr(), u32),
                                                 st["holders"]))
        cp._check(L.clairplan_export_holders(plan._h, ctypes.cast(h_off.data_ptr(), u64),
                                             ctypes.cast(h_hold.data_ptr(), u32), st["holders"]))

    step()
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    n = max(1, args.steps)
    t = time.perf_counter()
    for _ in range(n):
        step()
    torch.cuda.synchronize()
    t = (time.perf_counter() - t) / n
    tv = torch.tensor([t], dtype=torch.float64, device="cuda")
    if world > 1:
        torch.distributed.all_reduce(tv, op=torch.distributed.ReduceOp.MAX)
    t = float(tv[0])
    H = st["holders"]
    return {"value": A_all / t, "unit": UNIT, "ms_per_step": t * 1e3,
            "h2d_bytes_per_step": 8 * F,
            "d2h_bytes_per_step": 4 * st["accesses"] + 4 * H + 12 * H + 8 * (F + 1),
            "path": ("clairplan_build_export: sizes H2D + build + streams/class lists/holders D2H "
                     "(pinned buffers; the stream copy overlaps the rest of the build)" if world == 1
                     else "clairplan_set_sizes (pinned H2D) + sharded build + export_streams/"
                     "class_lists/holders (pinned D2H)"), "workers_per_rank": nloc}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", type=int, default=4, choices=sorted(CONFIGS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        run_reference(args, cfg)
    else:
        run_ours(args, cfg)


if __name__ == "__main__":
    main()
