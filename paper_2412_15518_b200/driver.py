"""SSP-RK3 hydro step driver on the device (the reference specifies the
step, but ships no driver: proj/tools/taskmesh_cli.cpp:1).

One step = [CFL dt on device] + 3 x (reference-exact ghost exchange ->
aggregated stage kernel over every leaf of the arena, in place, with the
rk3_combine epilogue, rk3.hpp:18-27).
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from ._lib import TmgpuError, lib
from .amr import Forest, unpack
from .hydro import SolverError


lib.tmgpu_forest_step_io.restype = C.c_int
lib.tmgpu_forest_step_io.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_double, C.c_double, C.c_double,
                                     C.c_int, C.c_void_p, C.POINTER(C.c_double), C.POINTER(TmgpuError)]
lib.tmgpu_forest_set_reflux.restype = C.c_int
lib.tmgpu_forest_set_reflux.argtypes = [C.c_void_p, C.c_int, C.POINTER(TmgpuError)]


class HydroDriver:
    def __init__(self, forest: Forest, gamma: float = 1.4, cfl: float = 0.4, fast: bool = False,
                 exact_ghosts: bool = False, reflux: bool = False):
        """exact_ghosts: reference 3-pass full-shell exchange (full ghosted arrays
        bitwise equal to the reference); default one-round face-only exchange
        (bitwise on every ghost the stage reads, hence on the state).
        reflux: flux-register correction at refinement jumps after every stage
        (flux_register.hpp:21-63 declared only; our restatement,
        oracle tmo_reflux_apply) — conserves mass across level jumps; on a
        distributed forest the fine face blocks of coarse leaves on other GPUs
        are exchanged after every stage (the same bits as one GPU)."""
        self.forest, self.gamma, self.cfl, self.fast = forest, gamma, cfl, fast
        self.exact_ghosts = exact_ghosts
        self.graph = True  # one GPU: the step replays as a cached CUDA graph (False: direct enqueue)
        self.steps = 0
        self.reflux = reflux
        if reflux:
            err = TmgpuError()
            _lib.check(lib.tmgpu_forest_set_reflux(forest.h, 1, C.byref(err)), err)

    def step(self, dt: float | None = None, stream=None, sync: bool = True, io=None) -> float | None:
        """Advance one SSP-RK3 step. dt None: CFL dt on the device. Returns
        the dt used (None when sync=False; errors are then latched until
        ``check``). io = (dev_in, dev_out): the step's input and/or output as
        compact interiors [local][V][E^3] in device memory (tensors or None) —
        scattered / gathered inside the step's own passes (tmgpu_forest_step_io)."""
        flags = ((_lib.TMGPU_FAST if self.fast else 0) | (0 if sync else _lib.TMGPU_ASYNC) |
                 (_lib.TMGPU_EXACT_GHOSTS if self.exact_ghosts else 0) |
                 (0 if self.graph else _lib.TMGPU_NO_GRAPH))
        used = C.c_double(0.0)
        err = TmgpuError()
        din, dout = io if io is not None else (None, None)
        rc = lib.tmgpu_forest_step_io(self.forest.h, None if din is None else din.data_ptr(),
                                      None if dout is None else dout.data_ptr(), float(dt or 0.0),
                                      self.cfl if dt is None else 0.0, self.gamma, flags, stream,
                                      C.byref(used), C.byref(err))
        _lib.check(rc, err, SolverError)
        self.steps += 1
        return used.value if sync else None

    def check(self, stream=None) -> None:
        err = TmgpuError()
        _lib.check(lib.tmgpu_forest_check(self.forest.h, stream, C.byref(err)), err, SolverError)

    def release_peers(self) -> None:
        """Collective: return a peer-memory forest to NCCL exchanges on every rank
        (amr.Forest.set_peer(False): barrier, unmap, barrier, free)."""
        if getattr(self.forest, "_peer", False):
            self.forest.set_peer(False)

    def regrid(self, refine=(), coarsen=()) -> None:
        """Refine then coarsen with the state carried along (Forest.regrid; on a
        distributed forest the collective dist.regrid, which re-partitions). Every
        face ghost is filled first (prolongation reads the parent's face ghosts)."""
        self.forest.fill_faces()
        if self.forest.local_count() != self.forest.leaf_count():
            from . import dist

            dist.regrid(self.forest, refine, coarsen)
        else:
            self.forest.regrid(refine, coarsen)
        if self.reflux:
            err = TmgpuError()
            _lib.check(lib.tmgpu_forest_set_reflux(self.forest.h, 1, C.byref(err)), err)


lib.tmgpu_stream_wait.restype = C.c_int
lib.tmgpu_stream_wait.argtypes = [C.c_void_p, C.c_void_p]
lib.tmgpu_forest_set_gravity_stream.restype = C.c_int
lib.tmgpu_forest_set_gravity_stream.argtypes = [C.c_void_p, C.c_void_p, C.POINTER(TmgpuError)]
lib.tmgpu_forest_set_gravity.restype = C.c_int
lib.tmgpu_forest_set_gravity.argtypes = [C.c_void_p, C.c_void_p, C.c_longlong, C.POINTER(TmgpuError)]


lib.tmgpu_forest_set_gravity_solver.restype = C.c_int
lib.tmgpu_forest_set_gravity_solver.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_void_p,
                                                C.c_void_p, C.c_void_p, C.c_void_p, C.c_longlong,
                                                C.POINTER(TmgpuError)]


class GravityHydroDriver(HydroDriver):
    """The gravity + hydro step of the metric (BASELINE.json): the SSP-RK3 hydro
    step with self-gravity from the AMR FMM (paper_2412_15518_b200.gravity.GravityAMR,
    our specification — the reference has no gravity), with the
    angular-momentum correction, as the stage kernel's source term (m += dt*rho*g,
    E += dt*rho*(v.g); oracle tmo_stage_subgrid_grav). The solves run inside the
    step (tmgpu_forest_set_gravity_solver):

      solves_per_step=3  (default) before every RK stage on that stage's input
                         state — the paper's coupling, one FMM iteration per
                         hydro iteration
      solves_per_step=6  the paper's count: per stage a second
                         solve on the stage's provisional density moves the
                         source to the trapezoid of the two fields
                         (csrc/grav_source.cu)
      solves_per_step=1  once per step on the initial state, held over the
                         three stages (round-1 behaviour)

    On a distributed forest (Forest.distribute) the solve is distributed as a
    locally essential tree with a multipole-moment exchange (GravityAMR.distribute);
    bitwise equal to one GPU. ``regrid`` refines/coarsens with the data carried
    along (Forest.regrid) and rebuilds the gravity plan (single GPU)."""

    def __init__(self, forest: Forest, gamma: float = 1.4, cfl: float = 0.4, fast: bool = False,
                 exact_ghosts: bool = False, am: bool = True, reflux: bool = False,
                 solves_per_step: int = 3):
        if solves_per_step not in (1, 3, 6):
            raise ValueError("solves_per_step must be 1, 3 or 6")
        super().__init__(forest, gamma, cfl, fast, exact_ghosts, reflux)
        self.am = am
        self.solves_per_step = solves_per_step
        self._setup_gravity()

    def _setup_gravity(self) -> None:
        import torch

        from .gravity import GravityAMR

        forest = self.forest
        leaves = np.array([unpack(int(p)) for p in forest.leaves()], dtype=np.int32).reshape(-1, 4)
        self.gravity = GravityAMR(leaves)
        comm = getattr(forest, "_comm", None)
        if forest.local_count() != forest.leaf_count():
            if comm is None:
                raise ValueError("distributed forest without a communicator")
            # its own NCCL communicator: the moment exchange runs on the gravity
            # stream concurrently with the hydro step's dt reduction and halo
            from .dist import Comm

            self.gcomm = Comm.from_torch()
            self.gravity.distribute(self.gcomm, forest._owner)
            self.moment_transport = "nccl"
            if getattr(forest, "_peer", False):  # the forest's halo is over peer memory
                try:  # collective; every rank agrees on the outcome
                    self.gravity.set_peer(True)
                    self.moment_transport = "peer"
                except (_lib.CudaError, RuntimeError) as ex:
                    self.moment_transport = f"nccl (peer setup failed: {ex})"
        # the solves run on a side stream, each overlapped with its stage's ghost
        # exchange (stage 1: also the CFL reduction; multi-GPU: the latency-bound
        # moment exchange); the stage kernel waits for it. TMGPU_GRAVITY_OVERLAP=0
        # keeps them on the step's stream (same results, bit for bit)
        import os

        self.gstream = None
        if os.environ.get("TMGPU_GRAVITY_OVERLAP", "1") != "0":
            self.gstream = torch.cuda.Stream(priority=-1)  # the critical path: first pick of SMs
            _lib.check(lib.tmgpu_forest_set_gravity_stream(forest.h, self.gstream.cuda_stream,
                                                           C.byref(TmgpuError())), TmgpuError())
        n = forest.local_count() * 512
        self.phi = torch.empty(n, dtype=torch.float64, device="cuda")
        self.g = torch.zeros(3 * n, dtype=torch.float64, device="cuda")
        six = self.solves_per_step == 6
        self.g2 = torch.zeros(3 * n, dtype=torch.float64, device="cuda") if six else None
        self.rho_tilde = torch.zeros(n, dtype=torch.float64, device="cuda") if six else None
        err = TmgpuError()
        _lib.check(lib.tmgpu_forest_set_gravity_solver(
            forest.h, self.gravity.h, self.solves_per_step, _lib.TMGPU_GRAV_AM if self.am else 0,
            self.phi.data_ptr(), self.g.data_ptr(), self.g2.data_ptr() if six else None,
            self.rho_tilde.data_ptr() if six else None, n, C.byref(err)), err)

    def solve_gravity(self, stream=None) -> None:
        """Enqueue one stand-alone solve on the current state into (phi, g)
        (the step solves by itself; this is for inspection)."""
        self.gravity.mass_from_arena(self.forest, stream)
        self.gravity.solve(None, am=self.am, phi=self.phi, g=self.g, stream=stream, sync=False)

    def regrid(self, refine=(), coarsen=()) -> None:
        """Refine then coarsen leaves with the state carried along (the
        reference's prolong_cell / restrict_cells, Forest.regrid; on a
        distributed forest the collective dist.regrid, which re-partitions), then
        rebuild the gravity plan and field for the new topology (and the reflux
        plan)."""
        self.close()
        if getattr(self, "moment_transport", "") == "peer":
            self.gravity.set_peer(False)  # collective, before the solver goes away
        self.forest.fill_faces()  # every face ghost valid: prolongation reads the parent's
        if self.forest.local_count() != self.forest.leaf_count():
            from . import dist

            dist.regrid(self.forest, refine, coarsen)
        else:
            self.forest.regrid(refine, coarsen)
        if self.reflux:
            err = TmgpuError()
            _lib.check(lib.tmgpu_forest_set_reflux(self.forest.h, 1, C.byref(err)), err)
        self._setup_gravity()

    def release_peers(self) -> None:
        """Collective on a distributed forest: tear the peer-memory exchanges down
        on every rank (barrier, unmap, barrier, free) before the forest or the
        solver is destroyed (freeing memory a peer still maps is undefined)."""
        self.close()
        if getattr(self, "moment_transport", "") == "peer":
            self.gravity.set_peer(False)
            self.moment_transport = "nccl"
        super().release_peers()

    def close(self) -> None:
        err = TmgpuError()
        lib.tmgpu_forest_set_gravity_solver(self.forest.h, None, 0, 0, None, None, None, None, 0,
                                            C.byref(err))
        lib.tmgpu_forest_set_gravity(self.forest.h, None, 0, C.byref(err))
        lib.tmgpu_forest_set_gravity_stream(self.forest.h, None, C.byref(err))


class HostStepPipeline:
    """Stepping from and to host (pinned) buffers with the transfers off the
    critical path: the host->device copy of step k+1's input runs on one copy
    stream while step k computes, the device->host copy of step k's result on a
    second copy stream while step k+1 computes (PCIe is full duplex). Device
    staging is double-buffered; CUDA events order every buffer reuse, so each
    step still moves its whole input in and its whole result out. The step
    itself reads the input staging buffer in its first pass and writes the output
    staging buffer from its last stage (tmgpu_forest_step_io).

        pipe = HostStepPipeline(GravityHydroDriver(forest))
        for _ in range(n):
            pipe.step(pin_in, pin_out)   # enqueue, returns at once
        pipe.synchronize()
    """

    def __init__(self, driver):
        import torch

        self.driver, self.forest = driver, driver.forest
        f = self.forest
        n = f.local_count() * f.vars * f.edge ** 3
        self.dev_in = [torch.empty(n, dtype=torch.float64, device="cuda") for _ in range(2)]
        self.dev_out = [torch.empty(n, dtype=torch.float64, device="cuda") for _ in range(2)]
        self.h2d, self.d2h = torch.cuda.Stream(), torch.cuda.Stream()
        self.compute = torch.cuda.current_stream()
        self.in_free, self.out_free = [None, None], [None, None]
        self.k = 0

    def step(self, pin_in, pin_out, dt: float | None = None) -> None:
        import torch

        b = self.k & 1
        cs = self.compute
        with torch.cuda.stream(self.h2d):
            if self.in_free[b] is not None:
                self.h2d.wait_event(self.in_free[b])
            self.dev_in[b].copy_(pin_in.reshape(-1), non_blocking=True)
            ev_in = torch.cuda.Event()
            ev_in.record(self.h2d)
        cs.wait_event(ev_in)
        if self.out_free[b] is not None:
            cs.wait_event(self.out_free[b])
        # the step reads its input straight from the staging buffer and its last
        # stage writes the output staging buffer (no separate scatter / gather)
        self.driver.step(dt, stream=cs.cuda_stream, sync=False, io=(self.dev_in[b], self.dev_out[b]))
        self.in_free[b] = torch.cuda.Event()
        self.in_free[b].record(cs)
        ev_out = torch.cuda.Event()
        ev_out.record(cs)
        with torch.cuda.stream(self.d2h):
            self.d2h.wait_event(ev_out)
            pin_out.reshape(-1).copy_(self.dev_out[b], non_blocking=True)
            self.out_free[b] = torch.cuda.Event()
            self.out_free[b].record(self.d2h)
        self.k += 1

    def synchronize(self) -> None:
        import torch

        torch.cuda.synchronize()
        self.driver.check()
