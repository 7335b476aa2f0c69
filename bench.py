#!/usr/bin/env python
"""Benchmark: sub-grid cell updates/s of the gravity + hydro step on B200.

Workload (BASELINE.json configs[2], the config the metric is quoted on):
rotating star on a 5-level AMR octree (leaf levels 2..5, 5,888 leaves of 8^3
cells = 3.01e6 cells). One step = the SSP-RK3 hydro step with self-gravity:
CFL dt + 3 x [adaptive FMM gravity solve on the stage's input state (the
angular-momentum correction included; our specification, DESIGN.md §7 — the
reference has no gravity code) || ghost exchange -> aggregated FP64 stage
kernel over every leaf with the gravity source + rk3 combine]. That is the
paper's coupling, one FMM iteration per hydro iteration;
--solves-per-step 6 runs the paper's count (a second solve per
stage on the provisional state), 1 the round-1 step (one solve held over the
stages).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--scenario star|dwd|sod|sedov] [--solves-per-step 1|3|6]

--scenario sod|sedov: BASELINE.json configs[3] (hydro-only, 6-level AMR);
dwd: configs[4] (7-level AMR). N>1 runs under torchrun, one rank per GPU;
the timed region is bracketed by a barrier + device synchronisation and the
max over ranks is reported. The reference arm (--impl reference) builds its
workload on the reference's own Tree (oracle/_ref/libtmref.so) and imports
nothing from the product.
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

METRIC = "sub-grid cell updates/sec (gravity+hydro step)"
UNIT = "cell-steps/s"
ALG_FLOP_PER_CELL = 633.25     # hydro stage FP64 ops per cell (div/sqrt = 1)
ALG_BYTES_PER_CELL = 180.0     # stage kernel, device-resident: 1280 staged cells x 40 B per
                               # 512 cells (100 B) + interior write 40 B + u0 read/write 40 B
# Gravity, FP64 flops per interaction, FMA = 2, geometry tabulated
# (per stencil offset for V, per distinct separation for W/X and U, built once
# with the plan). The order-2 Cartesian M2L is 28 multiply-adds; into a leaf
# patch only L0 and L_i are needed (22); a leaf-cell source has D = Q = 0, so
# its term is the monopole one: 1 mul + 1 add + 3 FMA into L0, L_i (8 flops),
# + 6 FMA into L_ij for an internal target (20). By (target, source) kind:
FLOP_M2L = {"ll": 8, "li": 44, "il": 20, "ii": 56}
FLOP_P2P, FLOP_P2P_U = 8, 8  # 4 FMA per same-depth or cross-depth pair


# scenario -> (kind, default min/max leaf level, bc, name)
SCENARIOS = {
    "star": (0, 2, 5, (0, 0, 0), "configs[2]: rotating star"),
    "dwd": (1, 2, 7, (0, 0, 0), "configs[4]: double-white-dwarf initial model (geometric refinement)"),
    "sod": (2, 2, 6, (0, 1, 1), "configs[3]: Sod shock tube (periodic x, reflective y/z)"),
    "sedov": (3, 2, 6, (0, 0, 0), "configs[3]: Sedov blast (E0 = 1 in the 8 central cells)"),
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--fast", action="store_true", help="FMA/reciprocal kernels (1e-10 parity)")
    ap.add_argument("--min-level", type=int, default=None)
    ap.add_argument("--max-level", type=int, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-steps", type=int, default=1)
    ap.add_argument("--cpu-budget", type=float, default=150.0,
                    help="reference arm: stop timing steps after this many seconds")
    ap.add_argument("--hydro-only", action="store_true", help="time the hydro step alone")
    ap.add_argument("--reflux", action="store_true",
                    help="flux-register correction at level jumps after every stage (SPEC.md:485; "
                         "across GPUs too); off by default: the reference's composed step has none")
    ap.add_argument("--solves-per-step", type=int, choices=[1, 3, 6], default=3,
                    help="FMM solves per step: 3 = one per RK stage (default), 6 = the paper's "
                         "count, 1 = once per step")
    ap.add_argument("--halo", choices=["nccl", "peer"], default="peer",
                    help="N>1 ghost-slab transport: NCCL send/recv or peer-memory stores")
    ap.add_argument("--scenario", choices=list(SCENARIOS), default="star")
    a = ap.parse_args()
    kind, lo, hi, bc, _ = SCENARIOS[a.scenario]
    a.min_level = lo if a.min_level is None else a.min_level
    a.max_level = hi if a.max_level is None else a.max_level
    a.kind, a.bc = kind, bc
    if a.scenario in ("sod", "sedov"):
        a.hydro_only = True  # configs[3] is hydro-only
    return a


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

    f = amr.build_scenario(amr.Scenario(args.kind), args.min_level, args.max_level, 0.1, bc=args.bc)
    state = f.scenario_state(amr.Scenario(args.kind))
    return f, state


def step_text(args):
    if args.hydro_only:
        return "SSP-RK3 hydro step: CFL dt + 3 x (ghost exchange + aggregated stage + rk3 combine)"
    sps = args.solves_per_step
    how = {1: "1 adaptive FMM solve per step (on the initial state, held over the 3 stages)",
           3: "3 adaptive FMM solves per step (one per RK stage on its input state, PAPER.md:240)",
           6: "6 adaptive FMM solves per step (the paper's count, PAPER.md:241: per stage on its "
              "input state + on its provisional state, trapezoid source)"}[sps]
    return ("gravity+hydro step: " + how + " (V/W/X/U lists, angular-momentum correction) + SSP-RK3 "
            "hydro step with the gravity source in the stage epilogue: CFL dt + 3 x (ghost exchange + "
            "aggregated stage + rk3 combine)")


def workload_config(n, args, extra=None):
    name = SCENARIOS[args.scenario][4]
    cfg = {"workload": f"{name}, {args.max_level}-level AMR octree "
                       f"(leaf levels {args.min_level}-{args.max_level}), {n} leaves x 8^3 cells, "
                       f"{step_text(args)}",
           "leaves": n, "cells": n * 512, "subgrid": "8^3 + 2 ghost layers, 5 vars (Euler)",
           "solves_per_step": 0 if args.hydro_only else args.solves_per_step,
           "reflux": bool(getattr(args, "reflux", False)),
           "l2": "inputs larger than L2 (ghosted arena %.0f MB > 126 MB L2)" % (n * 69120 / 1e6),
           "parity": ("hydro: fast <=1e-10 scaled vs reference" if args.fast else
                      "hydro: bitwise vs the reference build (tests/test_forest_gpu.py)") +
                     ("" if args.hydro_only else
                      "; gravity+hydro: bitwise vs the oracle composition at this size "
                      "(tests/test_gravity_c3_gpu.py, tests/test_gravity_hydro_gpu.py)")}
    if extra:
        cfg.update(extra)
    return cfg


def time_reference(args, steps, warmup=0, budget_s=None):
    """The CPU step on the host cores, entirely on the reference side: the
    workload is built on the reference's own Tree (oracle/ref_capi.cpp
    tmref_tree_scenario/_fill, the same leaves and bits as the GPU arm's,
    tests/test_forest.py), and one step is tmref_gravity_hydro_step: the
    reference's hydro (fill_ghosts_sync single-threaded as in the reference,
    AggregationRegion(make_stage_kernel) over Scheduler(ncores), rk3_combine)
    with the CFL dt inside the call, plus — gravity, which the reference does
    not have — the patch-sparse CPU restatement of our FMM
    (oracle/gravity_amr_sparse.c: tabulated geometry, SIMD V lists, OpenMP;
    its topology plan built once, like the GPU's) at the same solves per step.
    Returns (median s/step, cores, mean phase seconds, steps timed, leaves, detail)."""
    # torchrun sets OMP_NUM_THREADS=1 in every process of a multi-process launch;
    # only rank 0 works here, so give the CPU path (its OpenMP FMM) all host
    # cores before the oracle library starts its thread pool
    os.environ["OMP_NUM_THREADS"] = str(os.cpu_count() or 1)
    from oracle import oracle as O

    ref = O.Ref()
    t = ref.tree(max_level=args.max_level, bc=args.bc)
    t.scenario(args.kind, args.min_level, args.max_level, 0.1)
    n = len(t.leaves())
    cores = os.cpu_count() or 1
    gravity = not args.hydro_only
    o = O.Oracle() if gravity else None
    g0 = time.perf_counter()
    plan = o.grav_plan(t.leaf_levels()) if gravity else None
    plan_s = time.perf_counter() - g0
    sps = args.solves_per_step if gravity else 0

    def one():
        w0 = time.perf_counter()
        _, secs = t.gravity_hydro_step(cfl=0.4, workers=cores, max_slices=8, solves_per_step=sps,
                                       plan=plan)
        return time.perf_counter() - w0, secs

    for _ in range(warmup):
        one()
    walls, tot = [], {}
    t_start = time.perf_counter()
    for _ in range(steps):
        w, secs = one()
        walls.append(w)
        for k, v in secs.items():
            tot[k] = tot.get(k, 0.0) + v
        if budget_s is not None and time.perf_counter() - t_start > budget_s:
            break
    k = len(walls)
    detail = {key: v / k for key, v in tot.items()}
    detail["gravity_plan_s"] = plan_s
    detail["fast_oracle"] = bool(o.fast) if o is not None else None
    return statistics.median(walls), cores, k, n, detail


def cpu_sample_text(steps, detail, cores, args):
    gravity = not args.hydro_only
    txt = (f"{steps} full step(s) of the same workload (built on the reference Tree) on {cores} host "
           f"threads: reference hydro (CFL dt {detail['cfl_s']:.3f} s, exchange {detail['exchange_s']:.2f} s "
           f"single-threaded as in the reference, stages {detail['stage_s']:.2f} s over {cores} workers)")
    if gravity:
        txt += (f" + gravity {detail['gravity_s']:.2f} s for {args.solves_per_step} solves (the patch-sparse "
                "CPU restatement of our FMM, oracle/gravity_amr_sparse.c: tabulated geometry, "
                f"{'AVX2 ' if detail.get('fast_oracle') else ''}SIMD V lists, OpenMP; plan built once in "
                f"{detail['gravity_plan_s']:.2f} s, untimed like the GPU's; the reference has no gravity code)")
    return txt


def fp64_peaks():
    """(DFMA, DMMA) FP64 TFLOP/s measured live by tools/probes/libtmprobe.so
    (diagnostics, not the product library; MEASURED_PEAKS.json has no FP64 entry)."""
    sys.path.insert(0, os.path.join(ROOT, "tools", "probes"))
    import probe

    return probe.fp64_peaks()


def hbm_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def profile_traffic(name):
    try:
        with open(os.path.join(ROOT, "profiles", name)) as fh:
            return json.load(fh)
    except Exception:
        return {}


# ---------------------------------------------------------------- arms
def run_reference_arm(args, rank, world):
    """The reference's CPU path on this box's host cores; rank 0 only. Imports
    nothing from the product (paper_2412_15518_b200)."""
    if rank != 0:
        return
    w = min(args.warmup, 1)
    sec, cores, k, n, detail = time_reference(args, args.steps, w, budget_s=args.cpu_budget)
    cells = n * 512
    v = cells / sec
    line = {"impl": "reference",
            "metric": METRIC if not args.hydro_only else "sub-grid cell updates/sec (hydro step)",
            "value": v, "unit": UNIT, "n_gpus": args.gpus, "steps": k, "warmup": w, "ms_per_step": sec * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": workload_config(n, args, {
                "reference": "hydro: oracle/_ref/libtmref.so (the unmodified taskmesh sources compiled in "
                             "place); workload built on the reference Tree (tmref_tree_scenario); gravity: "
                             "oracle/gravity_amr_sparse.c (no reference code exists)",
                "same_steps": k == args.steps,
                "steps_note": None if k == args.steps else
                f"stopped after {k} of {args.steps} steps (--cpu-budget {args.cpu_budget:.0f} s)"}),
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores,
                             "kind": "reference" if args.hydro_only else "reference+port",
                             "sample": cpu_sample_text(k, detail, cores, args)},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    if not args.hydro_only:  # the hydro part of the same steps
        hs = detail["cfl_s"] + detail["exchange_s"] + detail["stage_s"]
        line["hydro_only"] = {"value": cells / hs, "unit": UNIT, "s_per_step": hs,
                              "note": "CFL + exchange + stage time of the same steps (no gravity)"}
    print(json.dumps(line), flush=True)


def run_ours(args, rank, world):
    import ctypes as C

    import torch

    from paper_2412_15518_b200 import _lib
    from paper_2412_15518_b200.driver import GravityHydroDriver, HydroDriver

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
    halo = "nccl"
    if world > 1 and args.halo == "peer":
        try:  # collective; every rank agrees on the outcome
            f.set_peer(True)
            halo = "peer"
        except Exception as ex:  # noqa: BLE001 - reported in the JSON line
            halo = f"nccl (peer setup failed: {ex})"
    f.set_interior(state)
    local_cells = f.local_count() * 512
    gravity = not args.hydro_only
    if gravity:
        drv = GravityHydroDriver(f, fast=args.fast, solves_per_step=args.solves_per_step,
                                 reflux=args.reflux)
    else:
        drv = HydroDriver(f, fast=args.fast, reflux=args.reflux)
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

    # per-phase device timing (separate pass, CUDA events on the launching
    # stream): gravity phases per solve, stage kernel per launch
    _lib.lib.tmgpu_forest_set_timing.argtypes = [C.c_void_p, C.c_int, C.c_void_p]
    _lib.lib.tmgpu_forest_timing.argtypes = [C.c_void_p] + [C.POINTER(C.c_double)] * 3 + [
        C.POINTER(C.c_longlong)]
    _lib.lib.tmgpu_forest_set_timing(f.h, 1, None)
    if gravity:
        drv.gravity.set_timing(True)
    for _ in range(5):
        drv.step(stream=sp, sync=False)
    torch.cuda.synchronize()
    tc, te, ts, nst = C.c_double(), C.c_double(), C.c_double(), C.c_longlong()
    _lib.lib.tmgpu_forest_timing(f.h, C.byref(tc), C.byref(te), C.byref(ts), C.byref(nst))
    _lib.lib.tmgpu_forest_set_timing(f.h, 0, None)
    steps_t = max(nst.value, 1)
    stage_ms = ts.value / (3 * steps_t)          # one stage launch = all local leaves
    exch_ms = te.value / (3 * steps_t)
    cfl_ms = tc.value / steps_t
    grav_ms, work = {}, {}
    if gravity:
        tot, ns = drv.gravity.timing()
        drv.gravity.set_timing(False)
        grav_ms = {k: v / max(ns, 1) for k, v in tot.items()}  # per solve
        work = drv.gravity.work()
    sps = args.solves_per_step if gravity else 0

    peak_tf, peak_dmma = fp64_peaks()
    hbm, hbm_src = hbm_peak()
    stage_gbps = local_cells * ALG_BYTES_PER_CELL / (stage_ms * 1e-3) / 1e9
    stage_tf = local_cells * ALG_FLOP_PER_CELL / (stage_ms * 1e-3) / 1e12
    stage_prof = profile_traffic("stage_kernel_latest.json")
    stage_roof = {"bound": "hbm", "achieved": stage_gbps, "peak": hbm, "unit": "GB/s",
                  "frac": stage_gbps / hbm, "traffic": stage_prof.get("dram_bytes_per_launch"),
                  "peak_source": hbm_src,
                  "kernel": "stage_kernel<5,%s>" % ("true" if args.fast else "false"),
                  "alg_bytes_per_cell": ALG_BYTES_PER_CELL, "launch_ms": stage_ms,
                  "cells_per_launch": local_cells,
                  "fp64": {"achieved": stage_tf, "peak": peak_tf, "unit": "TFLOP/s",
                           "frac": stage_tf / peak_tf if peak_tf else None,
                           "peak_dmma": peak_dmma, "frac_vs_dmma": stage_tf / peak_dmma if peak_dmma else None,
                           "alg_flop_per_cell": ALG_FLOP_PER_CELL}}
    share = {"hydro_stage": 3 * stage_ms / ms, "hydro_exchange": 3 * exch_ms / ms,
             "hydro_cfl": cfl_ms / ms}
    if gravity:
        m2l_flop = sum((work["v_" + k] + work["wx_" + k]) * f for k, f in FLOP_M2L.items())
        # the three M2L kernels timed alone (the timing pass serialises them;
        # the timed steps overlap mono with the upward pass and the fused kernel)
        k_ms = {k: grav_ms["k_" + k] for k in ("mono", "fused", "wx")}
        m2l_ms = sum(k_ms.values())
        m2l_tf = m2l_flop / (m2l_ms * 1e-3) / 1e12
        wx_flop = sum(work["wx_" + k] * f for k, f in FLOP_M2L.items())
        mono_flop = work["v_mono"] * FLOP_M2L["ll"]
        k_flop = {"mono": mono_flop, "fused": m2l_flop - wx_flop - mono_flop, "wx": wx_flop}
        per_kernel = {k: {"ms": k_ms[k], "alg_flop": k_flop[k],
                          "tflops": k_flop[k] / (k_ms[k] * 1e-3) / 1e12 if k_ms[k] else None,
                          "frac": (k_flop[k] / (k_ms[k] * 1e-3) / 1e12 / peak_tf) if k_ms[k] and peak_tf else None}
                      for k in k_ms}
        m2l_prof = profile_traffic("m2l_kernel_latest.json")
        roofline = {"bound": "fp64", "achieved": m2l_tf, "peak": peak_tf, "unit": "TFLOP/s",
                    "frac": m2l_tf / peak_tf if peak_tf else None,
                    "peak_dmma": peak_dmma, "frac_vs_dmma": m2l_tf / peak_dmma if peak_dmma else None,
                    "traffic": m2l_prof.get("dram_bytes_per_launch"),
                    "kernel": "gravity M2L: amr_m2l_mono (leaf patches among leaf patches) + "
                              "amr_m2l_fused (the rest) + amr_wx (W/X lists), all levels",
                    "launch_ms": m2l_ms,
                    "launch_ms_note": "sum of the three kernels' durations, each timed alone between CUDA "
                                      "events on the solve's stream (a separate timing pass serialises them; "
                                      "the timed steps overlap mono with the upward pass)",
                    "per_kernel": per_kernel,
                    "alg_flop_per_launch": m2l_flop,
                    "alg_flop": "per V pair / W-X entry by (target, source) kind (l leaf, i internal): "
                                + ", ".join(f"{k} {f} x {work['v_' + k] + work['wx_' + k]}"
                                            for k, f in FLOP_M2L.items())
                                + " (FMA = 2; a leaf source's D, Q are zero)",
                    "peak_source": "live DFMA microbenchmark (tools/probes/libtmprobe.so "
                                   "tmgpu_fp64_peak; the M2L is DFMA code); peak_dmma = the FP64 "
                                   "tensor-core (DMMA m8n8k4) probe, the chip's FP64 ceiling "
                                   "(MEASURED_PEAKS.json has no FP64 entry)",
                    "launch_note": "one M2L launch per solve; %d solves per step" % sps,
                    "hydro_stage": stage_roof}
        for k, v in grav_ms.items():
            if not k.startswith("k_"):
                share["gravity_" + k] = sps * v / ms
        step_flop = (sps * (m2l_flop + work["p2p_pairs"] * FLOP_P2P + work["u_cross_entries"] * FLOP_P2P_U)
                     + 3 * local_cells * ALG_FLOP_PER_CELL)
        roofline["step_fp64"] = {"achieved": step_flop / (ms * 1e-3) / 1e12, "unit": "TFLOP/s",
                                 "frac": step_flop / (ms * 1e-3) / 1e12 / peak_tf if peak_tf else None,
                                 "note": "all algorithmic FP64 of the step / step time"}
    else:
        roofline = stage_roof
    roofline["step_share"] = share
    if gravity:
        roofline["step_share_note"] = (
            "device-event phase times (a timing pass with the M2L kernels serialised) x occurrences per "
            "step / step time; every gravity solve runs "
            "on its own stream concurrently with its stage's ghost exchange (stage 1: and the CFL "
            "reduction), whose interval includes the wait for it, so the shares overlap")
    roofline["gravity_work"] = work or None
    if dist:  # per-rank phase times (ms per step, device events): the load balance
        mine = {"cfl": cfl_ms, "exchange": 3 * exch_ms, "stage": 3 * stage_ms,
                **{"gravity_" + k: sps * v for k, v in grav_ms.items()}}
        ranks = [None] * world
        dist.all_gather_object(ranks, {k: round(v, 4) for k, v in mine.items()})
        roofline["phase_ms_by_rank"] = ranks

    # e2e through the public API with host buffers (pinned): every step moves
    # its whole input H2D and its whole result D2H; HostStepPipeline overlaps
    # step k+1's H2D and step k-1's D2H with step k's compute (copy streams,
    # double-buffered staging). Timed from the first H2D to the last D2H.
    from paper_2412_15518_b200.driver import HostStepPipeline

    pin_in = torch.from_numpy(np.ascontiguousarray(state)).pin_memory()
    pin_out = torch.empty_like(pin_in).pin_memory()
    pipe = HostStepPipeline(drv)
    for _ in range(2):
        pipe.step(pin_in, pin_out)
    pipe.synchronize()
    barrier()
    # steady-state throughput of the pipelined host->device->host stepping: the
    # interval between the completed D2H of step W and of step W + K. Every
    # step in it still copies its whole input in and its whole result out; the
    # one-time fill (first H2D) and drain (last compute + D2H) stay outside, as
    # for any pipelined stream of steps.
    k_e2e = max(10, args.steps)
    a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(2):
        pipe.step(pin_in, pin_out)
    a0.record(pipe.d2h)
    h0 = time.perf_counter()
    for _ in range(k_e2e):
        pipe.step(pin_in, pin_out)
    host_ms = (time.perf_counter() - h0) * 1e3 / k_e2e  # host time to enqueue one step (no sync)
    a1.record(pipe.d2h)
    pipe.synchronize()
    e2e_ms = a0.elapsed_time(a1) / k_e2e
    if dist:
        t = torch.tensor([e2e_ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    nbytes = state.nbytes

    # hydro-only step on the same forest and state (the gravity solver detached):
    # the number the reference's own hydro step is compared with
    hydro_only = None
    if gravity:
        drv.close()
        hdrv = HydroDriver(f, fast=args.fast)
        for _ in range(3):
            hdrv.step(stream=sp, sync=False)
        hdrv.check(stream=sp)
        barrier()
        kh = max(10, args.steps)
        h0, h1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        h0.record(stream)
        for _ in range(kh):
            hdrv.step(stream=sp, sync=False)
        h1.record(stream)
        barrier()
        hdrv.check(stream=sp)
        hms = h0.elapsed_time(h1) / kh
        if dist:
            t = torch.tensor([hms], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            hms = float(t.item())
        hydro_only = {"value": cells / (hms * 1e-3), "unit": UNIT, "ms_per_step": hms, "steps": kh,
                      "note": "the SSP-RK3 hydro step alone on the same forest (device-resident)"}

    line = {"metric": METRIC if gravity else "sub-grid cell updates/sec (hydro step)",
            "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong",
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (analytic %s, scenario.cpp; std::mt19937_64 density noise)" % args.scenario,
            "config": workload_config(n, args, {
                "parallelism": (f"leaves partitioned over {world} GPUs (partition_leaves, "
                                "contiguous Morton ranges); cross-GPU ghost slabs " +
                                ("packed straight into the receivers' buffers over NVLink (CUDA "
                                 "IPC peer memory, flag-word sync)" if halo == "peer" else
                                 "by grouped NCCL send/recv" + halo[4:]) + " per RK stage; dt by "
                                "ncclAllReduce(min)" +
                                ("; gravity: locally essential tree — owned-subtree upward pass, "
                                 "subtree-root and halo moments " +
                                 ("stored straight into the peers' moment arrays (CUDA IPC)"
                                  if getattr(drv, "moment_transport", "") == "peer" else
                                  "by NCCL all-gather + grouped send/recv " +
                                  getattr(drv, "moment_transport", "nccl")[4:]) +
                                 ", M2L/L2L/L2P on the owned subtree, every solve overlapped "
                                 "with its stage's ghost exchange" if gravity else ""))
                if world > 1 else "single GPU"}),
            "e2e": {"value": cells / (e2e_ms * 1e-3), "unit": UNIT,
                    "h2d_bytes_per_step": nbytes, "d2h_bytes_per_step": nbytes,
                    "ms_per_step": e2e_ms, "steps": k_e2e, "host_enqueue_ms_per_step": host_ms,
                    "path": "paper_2412_15518_b200.driver.HostStepPipeline(" + type(drv).__name__ +
                            ").step(pinned in, pinned out): H2D -> tmgpu_forest_step_io (input scattered "
                            "in the step's first pass, output written by its last stage) -> D2H, copies "
                            "overlapped with the neighbouring steps' compute",
                    "timing": "steady state: completed D2H of step W to that of step W + K (every step "
                              "copies its whole input in and result out; one-time fill/drain excluded)"},
            "roofline": roofline,
            "gpu_launches": launches,
            "clocks": clk.summary()}

    if hydro_only:
        line["hydro_only"] = hydro_only
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            sec, cores, k, _, detail = time_reference(args, args.cpu_steps, 0)
            line["cpu_baseline"] = {"value": cells / sec, "unit": UNIT, "cores": cores,
                                    "kind": "reference+port" if gravity else "reference",
                                    "sample": cpu_sample_text(k, detail, cores, args)}
            if hydro_only:
                hs = detail["cfl_s"] + detail["exchange_s"] + detail["stage_s"]
                hydro_only["cpu_reference_value"] = cells / hs
                hydro_only["ratio_vs_cpu_reference"] = hydro_only["value"] / (cells / hs)
        except Exception as ex:  # reference build missing on this box
            line["cpu_baseline"] = {"value": None, "unit": UNIT, "cores": 0, "kind": "reference",
                                    "sample": f"unavailable: {ex}"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:  # collective teardown of the peer-memory exchanges, then the group
        (hdrv if gravity else drv).release_peers()
        if gravity:
            drv.release_peers()
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
