#!/usr/bin/env python
"""Benchmark: sub-grid cell updates/s of the full SSP-RK3 hydro step on B200.

Workload (BASELINE.json configs[2], the config the metric is quoted on):
rotating star on a 5-level AMR octree (levels 2..5, 5,888 leaves of 8^3
cells = 3.01e6 cells), one step = CFL dt + 3 x [reference-exact ghost
exchange -> aggregated FP64 stage kernel over every leaf + rk3_combine].
Gravity has no reference implementation and is not in the
timed step yet.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N>1 runs under torchrun, one rank per GPU; the timed region is bracketed by
a barrier + device synchronisation and the max over ranks is reported.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "sub-grid cell updates/sec (hydro step; gravity+hydro step once gravity lands)"
UNIT = "cell-steps/s"
ALG_FLOP_PER_CELL = 633.25     # hydro stage FP64 ops per cell (div/sqrt = 1)
ALG_BYTES_PER_CELL = 180.0     # stage kernel, device-resident: 1280 staged cells x 40 B per
                               # 512 cells (100 B) + interior write 40 B + u0 read/write 40 B


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--fast", action="store_true", help="FMA/reciprocal kernels (1e-10 parity)")
    ap.add_argument("--min-level", type=int, default=2)
    ap.add_argument("--max-level", type=int, default=5)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-steps", type=int, default=2)
    ap.add_argument("--no-gravity", action="store_true")
    return ap.parse_args()


# ---------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md)."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.lines, self.proc = index, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        time.sleep(0.3)
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------- workload
def build_workload(args):
    from paper_2412_15518_b200 import amr

    f = amr.build_scenario(amr.Scenario.rotating_star, args.min_level, args.max_level, 0.1)
    state = f.scenario_state(amr.Scenario.rotating_star)
    return f, state


def workload_config(f, args, extra=None):
    n = f.leaf_count()
    cfg = {"workload": f"rotating star, {args.max_level}-level AMR octree "
                       f"(leaf levels {args.min_level}-{args.max_level}), {n} leaves x 8^3 cells, full "
                       "SSP-RK3 hydro step: CFL dt + 3 x (ghost exchange + aggregated stage + rk3 combine)",
           "leaves": n, "cells": n * 512, "subgrid": "8^3 + 2 ghost layers, 5 vars (Euler)",
           "l2": "inputs larger than L2 (ghosted arena %.0f MB > 126 MB L2)" % (n * 69120 / 1e6),
           "parity": "fast: <=1e-10 scaled vs reference" if args.fast else
                     "bitwise vs reference (tests/test_forest_gpu.py)"}
    if extra:
        cfg.update(extra)
    return cfg


def reference_setup(f, state):
    """The same topology + initial state inside the UNMODIFIED reference."""
    from oracle import oracle as O
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from helpers import interior_to_ghosted, replay_on_reference

    ref = O.Ref()
    t = replay_on_reference(ref, f, int(max(int(p) >> 60 for p in f.leaves())))
    g = interior_to_ghosted(state)
    for i, p in enumerate(f.leaves()):
        t.grid(int(p))[:] = g[i]
    return ref, t


def reference_dt(ref, t, f, cfl=0.4):
    h = ref.encode_header(1, 1.0, 0.0)
    return cfl * min(t.cell_size(int(p) >> 60) / ref.max_wavespeed(h, t.grid(int(p)).copy())
                     for p in f.leaves())


def time_reference(f, state, steps, warmup=0):
    """Reference CPU step(s) on the host cores: returns (s/step, cores, detail)."""
    ref, t = reference_setup(f, state)
    cores = os.cpu_count() or 1
    for _ in range(warmup):
        t.hydro_step(reference_dt(ref, t, f), workers=cores, max_slices=8)
    walls, ex, st = [], 0.0, 0.0
    for _ in range(steps):
        dt = reference_dt(ref, t, f)
        t0 = time.perf_counter()
        tex, tst = t.hydro_step(dt, workers=cores, max_slices=8)
        walls.append(time.perf_counter() - t0)
        ex += tex
        st += tst
    return statistics.median(walls), cores, {"exchange_s": ex / steps, "stage_s": st / steps}


M2L_FLOP = 68  # per interaction (oracle/gravity_oracle.c contraction, geometry tabulated)
P2P_FLOP = 20  # per near-field pair (sqrt and division counted as 1)


def fmm_work(D):
    """(M2L interactions, P2P pairs) of the FMM on level D."""
    def axis(n, lo, hi):
        return sum(sum(1 for d in range(lo(i), hi(i) + 1) if 0 <= i + d < n) for i in range(n))

    m2l = 0
    for l in range(2, D + 1):
        n = 1 << l
        A = axis(n, lambda i: -2 - (i & 1), lambda i: 3 - (i & 1))
        B = axis(n, lambda i: -1, lambda i: 1)
        m2l += A ** 3 - B ** 3
    n = 1 << D
    B = axis(n, lambda i: -1, lambda i: 1)
    return m2l, B ** 3 - n ** 3


def bench_gravity(stream, peak_tf):
    """configs[1]: uniform level-4 octree (4,096 leaves, 128^3 cells), one FMM
    gravity solve from the device arena (rho -> masses -> P2M..P2P)."""
    import torch

    from paper_2412_15518_b200 import amr
    from paper_2412_15518_b200.gravity import GravitySolver

    f = amr.build_scenario(amr.Scenario.rotating_star, 4, 4)
    f.alloc()
    f.set_interior(f.scenario_state(amr.Scenario.rotating_star))
    G = GravitySolver(7)
    n3 = 128 ** 3
    phi = torch.empty(n3, dtype=torch.float64, device="cuda")
    g = torch.empty(3 * n3, dtype=torch.float64, device="cuda")
    sp = stream.cuda_stream
    for _ in range(3):
        G.solve_forest(f, phi, g, stream=sp, sync=False)
    torch.cuda.synchronize()
    reps = 20
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(reps):
        G.solve_forest(f, phi, g, stream=sp, sync=False)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    m2l, p2p = fmm_work(7)
    tf = (m2l * M2L_FLOP + p2p * P2P_FLOP) / (ms * 1e-3) / 1e12
    return {"config": "configs[1]: rotating star, uniform level-4 octree (4,096 leaves, 128^3 "
                      "cells), one FMM solve (our spec, DESIGN.md §7; no reference exists)",
            "ms_per_solve": ms, "cells_per_s": n3 / (ms * 1e-3),
            "m2l_interactions": m2l, "p2p_pairs": p2p,
            "roofline": {"bound": "fp64", "achieved": tf, "peak": peak_tf, "unit": "TFLOP/s",
                         "frac": tf / peak_tf if peak_tf else None,
                         "alg_flop": f"{M2L_FLOP}/M2L interaction + {P2P_FLOP}/P2P pair"}}


# ---------------------------------------------------------------- arms
def run_reference_arm(args, rank, world):
    if rank != 0:
        return
    f, state = build_workload(args)
    cells = f.leaf_count() * 512
    # bounded: every reference step is seconds of CPU work; cap the timed steps
    k = max(1, min(args.steps, 5))
    w = min(args.warmup, 1)
    sec, cores, detail = time_reference(f, state, k, w)
    v = cells / sec
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": k, "warmup": w, "ms_per_step": sec * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(f, args, {"reference": "oracle/_ref/libtmref.so (unmodified "
                                                "taskmesh sources): fill_ghosts_sync + AggregationRegion"
                                                "(make_stage_kernel, W=1, max_slices=8) + rk3_combine"}),
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "reference",
                             "sample": f"{k} full C3 steps (requested {args.steps}), exchange "
                                       f"{detail['exchange_s']:.2f} s (single-threaded), stages "
                                       f"{detail['stage_s']:.2f} s over {cores} workers"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_ours(args, rank, world):
    import ctypes as C

    import torch

    from paper_2412_15518_b200 import _lib
    from paper_2412_15518_b200.driver import HydroDriver

    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    f, state = build_workload(args)
    n = f.leaf_count()
    cells = n * 512  # whole job
    if world > 1:  # leaves partitioned over the GPUs (partition_leaves), NCCL halos
        from paper_2412_15518_b200 import dist as tmdist

        owner = tmdist.partition(f, world)
        comm = tmdist.Comm.from_torch()
        f.distribute(comm, owner)
        lo, hi = tmdist.local_range(owner, rank)
        state = np.ascontiguousarray(state[lo:hi])
    f.alloc()
    f.set_interior(state)
    local_cells = f.local_count() * 512
    drv = HydroDriver(f, fast=args.fast)
    stream = torch.cuda.current_stream()
    sp = stream.cuda_stream

    def barrier():
        if dist:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        drv.step(stream=sp, sync=False)
    drv.check(stream=sp)
    barrier()
    l0 = _lib.launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        barrier()
        e0.record(stream)
        for _ in range(args.steps):
            drv.step(stream=sp, sync=False)
        e1.record(stream)
        barrier()
    launches = _lib.launch_count() - l0
    drv.check(stream=sp)
    ms = e0.elapsed_time(e1) / args.steps
    if dist:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = cells / (ms * 1e-3)

    # per-phase device timing (separate pass; kernel share of the step)
    err = _lib.TmgpuError()
    _lib.lib.tmgpu_forest_set_timing.argtypes = [C.c_void_p, C.c_int, C.c_void_p]
    _lib.lib.tmgpu_forest_timing.argtypes = [C.c_void_p] + [C.POINTER(C.c_double)] * 3 + [
        C.POINTER(C.c_longlong)]
    _lib.lib.tmgpu_forest_set_timing(f.h, 1, None)
    for _ in range(3):
        drv.step(stream=sp, sync=False)
    torch.cuda.synchronize()
    tc, te, ts, nst = C.c_double(), C.c_double(), C.c_double(), C.c_longlong()
    _lib.lib.tmgpu_forest_timing(f.h, C.byref(tc), C.byref(te), C.byref(ts), C.byref(nst))
    _lib.lib.tmgpu_forest_set_timing(f.h, 0, None)
    steps_t = max(nst.value, 1)
    stage_ms = ts.value / (3 * steps_t)          # one stage launch = all leaves
    exch_ms = te.value / (3 * steps_t)
    cfl_ms = tc.value / steps_t

    # FP64 peak: MEASURED_PEAKS.json has no FP64 entry -> DFMA microbenchmark
    peak_tf, pms = C.c_double(0), C.c_double(0)
    _lib.lib.tmgpu_fp64_peak.argtypes = [C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_double),
                                         C.c_void_p]
    _lib.lib.tmgpu_fp64_peak(20000, C.byref(peak_tf), C.byref(pms), None)
    hbm_peak = 6545.6
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            hbm_peak = float(json.load(fh)["hbm_gbs"])
    except Exception:
        pass
    gbps = local_cells * ALG_BYTES_PER_CELL / (stage_ms * 1e-3) / 1e9
    tflops = local_cells * ALG_FLOP_PER_CELL / (stage_ms * 1e-3) / 1e12
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "stage_kernel_latest.json")) as fh:
            prof = json.load(fh)
            traffic = prof.get("dram_bytes_per_launch")
    except Exception:
        prof = {}

    # e2e through the public API with host buffers (pinned), per step:
    # H2D of the state, one step, D2H of the updated state.
    pin_in = torch.from_numpy(np.ascontiguousarray(state)).pin_memory()
    pin_out = torch.empty_like(pin_in).pin_memory()
    f.set_interior(pin_in)
    drv.step(stream=sp)
    barrier()
    e2 = []
    for _ in range(max(3, min(args.steps, 10))):
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record(stream)
        f.set_interior(pin_in)
        drv.step(stream=sp, sync=False)
        f.get_interior(pin_out)
        a1.record(stream)
        torch.cuda.synchronize()
        e2.append(a0.elapsed_time(a1))
    e2e_ms = statistics.median(e2)
    if dist:
        t = torch.tensor([e2e_ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    nbytes = state.nbytes

    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (analytic rotating star + "
            "1e-3 density noise, std::mt19937_64)",
            "config": workload_config(f, args, {
                "parallelism": (f"leaves partitioned over {world} GPUs (partition_leaves, "
                                "contiguous Morton ranges); cross-GPU ghost slabs by grouped "
                                "NCCL send/recv per RK stage; dt by ncclAllReduce(min)")
                if world > 1 else "single GPU"}),
            "e2e": {"value": cells / (e2e_ms * 1e-3), "unit": UNIT,
                    "h2d_bytes_per_step": nbytes, "d2h_bytes_per_step": nbytes,
                    "ms_per_step": e2e_ms,
                    "path": "paper_2412_15518_b200.amr.Forest.set_interior(pinned) -> "
                            "HydroDriver.step -> Forest.get_interior(pinned)"},
            "roofline": {"bound": "hbm", "achieved": gbps, "peak": hbm_peak, "unit": "GB/s",
                         "frac": gbps / hbm_peak, "traffic": traffic,
                         "kernel": "stage_kernel<5,%s>" % ("true" if args.fast else "false"),
                         "alg_bytes_per_cell": ALG_BYTES_PER_CELL,
                         "launch_ms": stage_ms, "cells_per_launch": local_cells,
                         "fp64": {"achieved": tflops, "peak": peak_tf.value, "unit": "TFLOP/s",
                                  "frac": tflops / peak_tf.value if peak_tf.value else None,
                                  "alg_flop_per_cell": ALG_FLOP_PER_CELL,
                                  "peak_source": "tmgpu_fp64_peak DFMA microbenchmark (live)"},
                         "fp64_pipe_util_ncu": prof.get("fp64_pipe_pct"),
                         "step_share": {"stage": 3 * stage_ms / ms, "exchange": 3 * exch_ms / ms,
                                        "cfl": cfl_ms / ms}},
            "gpu_launches": launches,
            "clocks": clk.summary()}

    if rank == 0 and world == 1 and not args.no_gravity:
        line["gravity"] = bench_gravity(stream, peak_tf.value)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            sec, cores, detail = time_reference(f, state, args.cpu_steps)
            line["cpu_baseline"] = {"value": cells / sec, "unit": UNIT, "cores": cores,
                                    "kind": "reference",
                                    "sample": f"{args.cpu_steps} full steps of the same workload "
                                              f"(exchange {detail['exchange_s']:.2f} s single-threaded, "
                                              f"stages {detail['stage_s']:.2f} s over {cores} threads)"}
        except Exception as ex:  # reference build missing on this box
            line["cpu_baseline"] = {"value": None, "unit": UNIT, "cores": 0, "kind": "reference",
                                    "sample": f"unavailable: {ex}"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.impl == "reference":
        run_reference_arm(args, rank, world)
    else:
        run_ours(args, rank, world)


if __name__ == "__main__":
    main()
