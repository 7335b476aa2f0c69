#!/usr/bin/env python
"""Benchmark: sub-grid cell updates/s of the gravity + hydro step on B200.

Workload (BASELINE.json configs[2], the config the metric is quoted on):
rotating star on a 5-level AMR octree (leaf levels 2..5, 5,888 leaves of 8^3
cells = 3.01e6 cells). One step = one adaptive FMM gravity solve with the
angular-momentum correction (our specification: the reference
has no gravity code) + the SSP-RK3 hydro step with the gravity source in the
stage epilogue: CFL dt + 3 x [ghost exchange -> aggregated FP64 stage kernel
over every leaf + rk3 combine].

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

METRIC = "sub-grid cell updates/sec (gravity+hydro step)"
UNIT = "cell-steps/s"
ALG_FLOP_PER_CELL = 633.25     # hydro stage FP64 ops per cell (div/sqrt = 1)
ALG_BYTES_PER_CELL = 180.0     # stage kernel, device-resident: 1280 staged cells x 40 B per
                               # 512 cells (100 B) + interior write 40 B + u0 read/write 40 B
# Gravity, FP64 flops per interaction, FMA = 2: the order-2
# Cartesian M2L is 28 multiply-adds once the geometry is known (into a leaf
# patch only L0 and L_i are needed: 22); W/X pairs also build their geometry
# (46 ops); same-depth P2P is 4 multiply-adds with tabulated geometry;
# cross-depth U pairs build theirs (15 ops).
FLOP_M2L_V, FLOP_M2L_V_LEAF, FLOP_M2L_WX, FLOP_P2P, FLOP_P2P_U = 56, 44, 102, 8, 23
FLOP_M2L_WX_LEAF = FLOP_M2L_WX - (FLOP_M2L_V - FLOP_M2L_V_LEAF)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--fast", action="store_true", help="FMA/reciprocal kernels (1e-10 parity)")
    ap.add_argument("--min-level", type=int, default=2)
    ap.add_argument("--max-level", type=int, default=5)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-steps", type=int, default=1)
    ap.add_argument("--hydro-only", action="store_true", help="time the hydro step alone")
    ap.add_argument("--halo", choices=["nccl", "peer"], default="peer",
                    help="N>1 ghost-slab transport: NCCL send/recv or peer-memory stores")
    ap.add_argument("--scenario", choices=["star", "dwd"], default="star",
                    help="star: configs[2] (default); dwd: configs[4] with --max-level 7")
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

    kind = amr.Scenario.rotating_star if args.scenario == "star" else amr.Scenario.double_white_dwarf
    f = amr.build_scenario(kind, args.min_level, args.max_level, 0.1)
    state = f.scenario_state(kind)
    return f, state


def workload_config(f, args, extra=None):
    n = f.leaf_count()
    step = ("SSP-RK3 hydro step: CFL dt + 3 x (ghost exchange + aggregated stage + rk3 combine)"
            if args.hydro_only else
            "gravity+hydro step: adaptive FMM solve (V/W/X/U lists, angular-momentum correction) "
            "+ SSP-RK3 hydro step with the gravity source in the stage epilogue: CFL dt + 3 x "
            "(ghost exchange + aggregated stage + rk3 combine)")
    name = ("configs[2]: rotating star" if args.scenario == "star" else
            "configs[4]: double-white-dwarf initial model (geometric refinement)")
    cfg = {"workload": f"{name}, {args.max_level}-level AMR octree "
                       f"(leaf levels {args.min_level}-{args.max_level}), {n} leaves x 8^3 cells, {step}",
           "leaves": n, "cells": n * 512, "subgrid": "8^3 + 2 ghost layers, 5 vars (Euler)",
           "l2": "inputs larger than L2 (ghosted arena %.0f MB > 126 MB L2)" % (n * 69120 / 1e6),
           "parity": ("hydro: fast <=1e-10 scaled vs reference" if args.fast else
                      "hydro: bitwise vs the reference build (tests/test_forest_gpu.py)") +
                     ("" if args.hydro_only else
                      "; gravity+hydro: bitwise vs the oracle composition (tests/test_gravity_hydro_gpu.py)")}
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


def time_reference(f, state, steps, warmup=0, gravity=True):
    """CPU step(s) on the host cores: the reference's own hydro step (the
    unmodified sources, oracle/_ref/libtmref.so: fill_ghosts_sync +
    AggregationRegion(make_stage_kernel) over Scheduler(ncores) + rk3_combine)
    and, for the gravity half (no reference code exists), our C restatement
    of the adaptive FMM (oracle/gravity_amr_oracle.c, OpenMP over targets) on
    the step's state. Returns (s/step, cores, detail)."""
    from oracle import oracle as O
    from paper_2412_15518_b200.gravity import forest_leaf_array

    ref, t = reference_setup(f, state)
    cores = os.cpu_count() or 1
    o = O.Oracle() if gravity else None
    lv = forest_leaf_array(f)
    h3 = (1.0 / (8.0 * 2.0 ** lv[:, 0].astype(np.float64))) ** 3

    def one():
        tg = 0.0
        if o is not None:
            ghosted = np.stack([t.grid(int(p)).reshape(5, 12, 12, 12)[0, 2:10, 2:10, 2:10].reshape(512)
                                for p in f.leaves()])
            g0 = time.perf_counter()
            o.grav_amr(lv, ghosted * h3[:, None], flags=1)
            tg = time.perf_counter() - g0
        dt = reference_dt(ref, t, f)
        h0 = time.perf_counter()
        tex, tst = t.hydro_step(dt, workers=cores, max_slices=8)
        return tg + time.perf_counter() - h0, tg, tex, tst

    for _ in range(warmup):
        one()
    walls, gr, ex, st = [], 0.0, 0.0, 0.0
    for _ in range(steps):
        w, tg, tex, tst = one()
        walls.append(w)
        gr += tg
        ex += tex
        st += tst
    return statistics.median(walls), cores, {"gravity_s": gr / steps, "exchange_s": ex / steps,
                                             "stage_s": st / steps}


def cpu_sample_text(steps, detail, cores, gravity=True):
    txt = (f"{steps} full step(s) of the same workload on {cores} host threads: reference hydro "
           f"(exchange {detail['exchange_s']:.2f} s single-threaded as in the reference, stages "
           f"{detail['stage_s']:.2f} s over {cores} workers)")
    if gravity:
        txt += (f" + gravity {detail['gravity_s']:.2f} s (our C restatement of the FMM, OpenMP; "
                "the reference has no gravity code)")
    return txt


def fp64_peak():
    """FP64 peak: MEASURED_PEAKS.json has no FP64 entry -> live DFMA microbenchmark."""
    import ctypes as C

    from paper_2412_15518_b200 import _lib

    peak_tf, pms = C.c_double(0), C.c_double(0)
    _lib.lib.tmgpu_fp64_peak.argtypes = [C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_double),
                                         C.c_void_p]
    _lib.lib.tmgpu_fp64_peak(20000, C.byref(peak_tf), C.byref(pms), None)
    return peak_tf.value


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
    if rank != 0:
        return
    f, state = build_workload(args)
    cells = f.leaf_count() * 512
    # bounded: every CPU step is seconds of work; cap the timed steps
    k = max(1, min(args.steps, 2))
    w = min(args.warmup, 1)
    sec, cores, detail = time_reference(f, state, k, w, gravity=not args.hydro_only)
    v = cells / sec
    line = {"impl": "reference", "metric": METRIC if not args.hydro_only else
            "sub-grid cell updates/sec (hydro step)", "value": v, "unit": UNIT,
            "n_gpus": args.gpus, "steps": k, "warmup": w, "ms_per_step": sec * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": workload_config(f, args, {"reference": "hydro: oracle/_ref/libtmref.so (the "
                                                "unmodified taskmesh sources compiled in place); gravity: "
                                                "oracle/gravity_amr_oracle.c (no reference code exists)"}),
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores,
                             "kind": "reference" if args.hydro_only else "reference+port",
                             "sample": cpu_sample_text(k, detail, cores, not args.hydro_only)},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
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
    full_state = state
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
        drv = GravityHydroDriver(f, fast=args.fast)
    else:
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
        grav_ms = {k: v / max(ns, 1) for k, v in tot.items()}
        work = drv.gravity.work()

    peak_tf = fp64_peak()
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
                           "alg_flop_per_cell": ALG_FLOP_PER_CELL}}
    share = {"hydro_stage": 3 * stage_ms / ms, "hydro_exchange": 3 * exch_ms / ms,
             "hydro_cfl": cfl_ms / ms}
    if gravity:
        m2l_flop = ((work["v_pairs"] - work["v_pairs_leaf"]) * FLOP_M2L_V +
                    work["v_pairs_leaf"] * FLOP_M2L_V_LEAF +
                    (work["wx_entries"] - work["wx_entries_leaf"]) * FLOP_M2L_WX +
                    work["wx_entries_leaf"] * FLOP_M2L_WX_LEAF)
        m2l_tf = m2l_flop / (grav_ms["m2l"] * 1e-3) / 1e12
        m2l_prof = profile_traffic("m2l_kernel_latest.json")
        roofline = {"bound": "fp64", "achieved": m2l_tf, "peak": peak_tf, "unit": "TFLOP/s",
                    "frac": m2l_tf / peak_tf if peak_tf else None,
                    "traffic": m2l_prof.get("dram_bytes_per_launch"),
                    "kernel": "amr_m2l (gravity M2L: V-list stencil + W/X lists), all levels",
                    "launch_ms": grav_ms["m2l"], "alg_flop_per_launch": m2l_flop,
                    "alg_flop": f"{FLOP_M2L_V}/V pair into internal patches, {FLOP_M2L_V_LEAF} into leaf "
                                f"patches ({work['v_pairs']} pairs, {work['v_pairs_leaf']} into leaves) + "
                                f"{FLOP_M2L_WX}/{FLOP_M2L_WX_LEAF} per W-X entry ({work['wx_entries']}) "
                                "(FMA = 2)",
                    "peak_source": "tmgpu_fp64_peak DFMA microbenchmark (live; MEASURED_PEAKS.json "
                                   "has no FP64 entry)",
                    "hydro_stage": stage_roof}
        for k, v in grav_ms.items():
            share["gravity_" + k] = v / ms
        step_flop = (m2l_flop + work["p2p_pairs"] * FLOP_P2P + work["u_cross_entries"] * FLOP_P2P_U
                     + 3 * local_cells * ALG_FLOP_PER_CELL)
        roofline["step_fp64"] = {"achieved": step_flop / (ms * 1e-3) / 1e12, "unit": "TFLOP/s",
                                 "frac": step_flop / (ms * 1e-3) / 1e12 / peak_tf if peak_tf else None,
                                 "note": "all algorithmic FP64 of the step / step time"}
    else:
        roofline = stage_roof
    roofline["step_share"] = share
    if gravity:
        roofline["step_share_note"] = (
            "device-event phase times / step time; the gravity solve runs on its own stream "
            "concurrently with the CFL reduction and the first ghost exchange, whose interval "
            "includes the wait for it, so the shares overlap")
    roofline["gravity_work"] = work or None
    if dist:  # per-rank phase times (ms per step, device events): the load balance
        mine = {"cfl": cfl_ms, "exchange": 3 * exch_ms, "stage": 3 * stage_ms,
                **{"gravity_" + k: v for k, v in grav_ms.items()}}
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
    k_e2e = max(5, args.steps)  # steady state: pipeline fill and drain amortised over K steps
    a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a0.record(pipe.h2d)
    for _ in range(k_e2e):
        pipe.step(pin_in, pin_out)
    a1.record(pipe.d2h)
    pipe.synchronize()
    e2e_ms = a0.elapsed_time(a1) / k_e2e
    if dist:
        t = torch.tensor([e2e_ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    nbytes = state.nbytes

    line = {"metric": METRIC if gravity else "sub-grid cell updates/sec (hydro step)",
            "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (analytic rotating star + "
            "1e-3 density noise, std::mt19937_64)",
            "config": workload_config(f, args, {
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
                                 ", M2L/L2L/L2P on the owned subtree, solve overlapped "
                                 "with the CFL reduction and first ghost exchange" if gravity else ""))
                if world > 1 else "single GPU"}),
            "e2e": {"value": cells / (e2e_ms * 1e-3), "unit": UNIT,
                    "h2d_bytes_per_step": nbytes, "d2h_bytes_per_step": nbytes,
                    "ms_per_step": e2e_ms, "steps": k_e2e,
                    "path": "paper_2412_15518_b200.driver.HostStepPipeline(" + type(drv).__name__ +
                            ").step(pinned in, pinned out): H2D -> Forest.set_interior -> step -> "
                            "Forest.get_interior -> D2H, copies overlapped with the neighbouring "
                            "steps' compute"},
            "roofline": roofline,
            "gpu_launches": launches,
            "clocks": clk.summary()}

    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            sec, cores, detail = time_reference(f, full_state, args.cpu_steps, gravity=gravity)
            line["cpu_baseline"] = {"value": cells / sec, "unit": UNIT, "cores": cores,
                                    "kind": "reference+port" if gravity else "reference",
                                    "sample": cpu_sample_text(args.cpu_steps, detail, cores, gravity)}
        except Exception as ex:  # reference build missing on this box
            line["cpu_baseline"] = {"value": None, "unit": UNIT, "cores": 0, "kind": "reference",
                                    "sample": f"unavailable: {ex}"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if gravity and hasattr(drv, "close"):
        drv.close()
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
