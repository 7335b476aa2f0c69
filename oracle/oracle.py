"""TEST INFRASTRUCTURE ONLY — ctypes access to the checkers.

Two CPU checkers live here, both built by ``oracle/Makefile``:

* ``Ref``    — the UNMODIFIED reference mini-app (``/root/reference/proj``)
  compiled in place into ``oracle/_ref/libtmref.so`` with the extern "C"
  shim ``oracle/ref_capi.cpp``. This is ground truth.
* ``Oracle`` — our plain-C restatement ``oracle/tm_oracle.c``
  (``oracle/_ref/liboracle.so``), pinned bitwise against ``Ref`` by
  ``tests/test_oracle_pin.py``.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
cpu_baseline / ``--impl reference`` legs may import this module. The
product (``paper_2412_15518_b200``) never does.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_DIR = os.path.join(HERE, "_ref")

_dp = C.POINTER(C.c_double)
_u64p = C.POINTER(C.c_uint64)
_i64p = C.POINTER(C.c_int64)
_ip = C.POINTER(C.c_int)


def dptr(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(_dp)


def u64ptr(a: np.ndarray):
    assert a.dtype == np.uint64 and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(_u64p)


def build(quiet: bool = True) -> None:
    """Build the checkers (needs /root/reference for the Ref part)."""
    import subprocess

    targets = ["oracle"]
    if os.path.isdir("/root/reference/proj"):
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", HERE, *targets], check=True,
                   stdout=subprocess.DEVNULL if quiet else None)


def ref_available() -> bool:
    return os.path.exists(os.path.join(REF_DIR, "libtmref.so"))


def oracle_available() -> bool:
    return os.path.exists(os.path.join(REF_DIR, "liboracle.so"))


class _Lib:
    def __init__(self, name: str):
        path = os.path.join(REF_DIR, name)
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} not built (run make -C oracle)")
        self.lib = C.CDLL(path)


class Ref(_Lib):
    """The reference's own code through oracle/ref_capi.cpp."""

    def __init__(self):
        super().__init__("libtmref.so")
        L = self.lib
        L.tmref_stage_fused.argtypes = [_dp, _dp, C.c_size_t, C.c_size_t, C.c_size_t,
                                        C.c_int, C.c_int, C.c_int, C.c_uint, C.c_char_p,
                                        C.c_size_t]
        L.tmref_in_slice.restype = C.c_size_t
        L.tmref_in_slice.argtypes = [C.c_int] * 3
        L.tmref_out_slice.restype = C.c_size_t
        L.tmref_out_slice.argtypes = [C.c_int] * 3
        L.tmref_encode_header.argtypes = [C.c_int] + [C.c_double] * 6 + [_dp]
        L.tmref_max_wavespeed.restype = C.c_double
        L.tmref_max_wavespeed.argtypes = [_dp, C.c_int, C.c_int, C.c_int, _dp]
        L.tmref_rk3_combine.restype = C.c_double
        L.tmref_rk3_combine.argtypes = [C.c_int, C.c_double, C.c_double]
        for f in ("tmref_minmod_scalar", "tmref_minmod_lane"):
            getattr(L, f).restype = C.c_double
            getattr(L, f).argtypes = [C.c_double, C.c_double]
        L.tmref_reconstruct_face.argtypes = [C.c_double] * 4 + [_dp]
        L.tmref_rusanov_euler.argtypes = [_dp, _dp, C.c_double, C.c_int, _dp]
        L.tmref_rusanov_scalar.restype = C.c_double
        L.tmref_rusanov_scalar.argtypes = [C.c_double] * 3
        L.tmref_morton_encode.argtypes = [C.c_int, C.c_uint64, C.c_uint64, C.c_uint64, _u64p]
        L.tmref_morton_decode.argtypes = [C.c_int, C.c_uint64, _u64p]
        L.tmref_morton_dfs_rank.restype = C.c_uint64
        L.tmref_morton_dfs_rank.argtypes = [C.c_int, C.c_uint64]
        L.tmref_partition_leaves.argtypes = [_u64p, C.c_size_t, C.c_int, _ip]
        L.tmref_prolong_cell.argtypes = [C.c_double] * 7 + [_dp]
        L.tmref_tree_create.restype = C.c_void_p
        L.tmref_tree_create.argtypes = [C.c_int] * 4 + [_ip, _ip]
        L.tmref_tree_destroy.argtypes = [C.c_void_p]
        L.tmref_tree_refine.argtypes = [C.c_void_p, C.c_uint64]
        L.tmref_tree_is_leaf.argtypes = [C.c_void_p, C.c_uint64]
        L.tmref_gravity_hydro_step.argtypes = [C.c_void_p, C.c_double, C.c_double, C.c_double, C.c_uint,
                                               C.c_size_t, C.c_int, C.c_void_p, C.c_void_p, C.c_int,
                                               _dp, _dp, C.c_char_p, C.c_size_t]
        L.tmref_tree_scenario.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_double]
        L.tmref_tree_scenario_fill.argtypes = [C.c_void_p, C.c_int, C.c_uint64]
        L.tmref_tree_coarsen.argtypes = [C.c_void_p, C.c_uint64]
        L.tmref_tree_leaves.restype = C.c_size_t
        L.tmref_tree_leaves.argtypes = [C.c_void_p, _u64p, C.c_size_t]
        L.tmref_tree_grid.restype = _dp
        L.tmref_tree_grid.argtypes = [C.c_void_p, C.c_uint64]
        L.tmref_tree_fill_ghosts.argtypes = [C.c_void_p]
        L.tmref_tree_flag.argtypes = [C.c_void_p, C.c_uint64, C.c_double]
        L.tmref_tree_balanced.argtypes = [C.c_void_p]
        L.tmref_tree_cell_size.restype = C.c_double
        L.tmref_tree_cell_size.argtypes = [C.c_void_p, C.c_int]
        L.tmref_tree_cell_center.argtypes = [C.c_void_p, C.c_uint64, C.c_int, C.c_int, C.c_int, _dp]
        L.tmref_tree_face_neighbor.argtypes = [C.c_void_p, C.c_uint64, C.c_int, C.c_int, _u64p, _ip]
        L.tmref_tree_plan.restype = C.c_size_t
        L.tmref_tree_plan.argtypes = [C.c_void_p, C.c_int, _i64p, C.c_size_t]
        L.tmref_hydro_step.argtypes = [C.c_void_p, C.c_double, C.c_double, C.c_uint, C.c_uint,
                                       C.c_size_t, _dp, _dp, C.c_char_p, C.c_size_t]
        L.tmref_stage_aggregated.restype = C.c_double
        L.tmref_stage_aggregated.argtypes = [_dp, C.c_size_t, C.c_int, C.c_int, C.c_int,
                                             C.c_uint, C.c_uint, C.c_size_t, _dp]

    # -- hydro
    def stage_fused(self, packed_in, count, edge=8, ghost=2, vars=5, lane_width=1):
        L = self.lib
        ins, outs = L.tmref_in_slice(edge, ghost, vars), L.tmref_out_slice(edge, ghost, vars)
        out = np.zeros(count * outs)
        err = C.create_string_buffer(256)
        rc = L.tmref_stage_fused(dptr(packed_in), dptr(out), ins, outs, count, edge, ghost,
                                 vars, lane_width, err, 256)
        return rc, out, err.value.decode()

    def encode_header(self, mode, dx, dt, gamma=1.4, advect=(1.0, 0.0, 0.0)):
        h = np.zeros(8)
        self.lib.tmref_encode_header(mode, dx, dt, gamma, *advect, dptr(h))
        return h

    def max_wavespeed(self, header, ghosted, edge=8, ghost=2, vars=5):
        return self.lib.tmref_max_wavespeed(dptr(header), edge, ghost, vars,
                                            dptr(ghosted) if ghosted is not None else None)

    # -- tree
    def tree(self, edge=8, ghost=2, vars=5, max_level=10, root_dims=(1, 1, 1), bc=(0, 0, 0)):
        return RefTree(self, edge, ghost, vars, max_level, root_dims, bc)


class RefTree:
    def __init__(self, ref: Ref, edge, ghost, vars, max_level, root_dims, bc):
        self.ref, self.L = ref, ref.lib
        self.edge, self.ghost, self.vars = edge, ghost, vars
        self.stride = edge + 2 * ghost
        rd = (C.c_int * 3)(*root_dims)
        b = (C.c_int * 3)(*bc)
        self.h = self.L.tmref_tree_create(edge, ghost, vars, max_level, rd, b)

    def __del__(self):
        if getattr(self, "h", None):
            self.L.tmref_tree_destroy(self.h)
            self.h = None

    def refine(self, packed: int) -> None:
        if self.L.tmref_tree_refine(self.h, packed) != 0:
            raise RuntimeError("reference refine failed")

    def coarsen(self, packed: int) -> None:
        if self.L.tmref_tree_coarsen(self.h, packed) != 0:
            raise RuntimeError("reference coarsen failed")

    def is_leaf(self, packed: int) -> bool:
        return bool(self.L.tmref_tree_is_leaf(self.h, packed))

    def scenario(self, kind: int, min_level: int, max_level: int, theta: float = 0.1,
                 seed: int = 2412518) -> None:
        """Build a BASELINE.json scenario on the reference Tree (ref_capi.cpp
        tmref_tree_scenario / _fill): 0 star, 1 DWD, 2 Sod, 3 Sedov."""
        if self.L.tmref_tree_scenario(self.h, kind, min_level, max_level, theta) != 0:
            raise RuntimeError("reference scenario refine failed")
        if self.L.tmref_tree_scenario_fill(self.h, kind, seed) != 0:
            raise RuntimeError("reference scenario fill failed")

    def leaf_levels(self) -> np.ndarray:
        """[n, 4] (level, I, J, K) of the leaves in leaves() order (NodeId::unpack,
        octree.hpp:35-41)."""
        p = self.leaves()
        return np.stack([(p >> np.uint64(60)), (p >> np.uint64(40)) & np.uint64(0xFFFFF),
                         (p >> np.uint64(20)) & np.uint64(0xFFFFF), p & np.uint64(0xFFFFF)],
                        axis=1).astype(np.int32)

    def leaves(self) -> np.ndarray:
        n = self.L.tmref_tree_leaves(self.h, None, 0)
        out = np.zeros(n, dtype=np.uint64)
        self.L.tmref_tree_leaves(self.h, u64ptr(out), n)
        return out

    def grid(self, packed: int) -> np.ndarray:
        p = self.L.tmref_tree_grid(self.h, packed)
        S = self.stride
        n = self.vars * S * S * S
        return np.ctypeslib.as_array(p, shape=(n,))

    def fill_ghosts(self) -> None:
        self.L.tmref_tree_fill_ghosts(self.h)

    def flag(self, packed: int, theta: float) -> bool:
        return bool(self.L.tmref_tree_flag(self.h, packed, theta))

    def balanced(self) -> bool:
        return bool(self.L.tmref_tree_balanced(self.h))

    def cell_size(self, level: int) -> float:
        return self.L.tmref_tree_cell_size(self.h, level)

    def face_neighbor(self, packed, axis, direction):
        ids = np.zeros(4, dtype=np.uint64)
        cnt = C.c_int(0)
        kind = self.L.tmref_tree_face_neighbor(self.h, packed, axis, direction, u64ptr(ids),
                                               C.byref(cnt))
        return kind, [int(x) for x in ids[: cnt.value]]

    def plan(self, axis) -> np.ndarray:
        n = self.L.tmref_tree_plan(self.h, axis, None, 0)
        rows = np.zeros((n, 7), dtype=np.int64)
        self.L.tmref_tree_plan(self.h, axis, rows.ctypes.data_as(_i64p), n)
        return rows

    def gravity_hydro_step(self, dt=0.0, cfl=0.4, gamma=1.4, workers=1, max_slices=8,
                           solves_per_step=0, plan=None, grav_flags=1):
        """The bench's CPU step (ref_capi.cpp tmref_gravity_hydro_step): the
        reference's hydro + `plan` (an Oracle GravPlan, the patch-sparse FMM)
        per the cadence; cfl > 0 computes dt inside. Returns (dt, seconds dict)."""
        secs = (C.c_double * 4)()
        used = C.c_double(0)
        err = C.create_string_buffer(256)
        fn = C.cast(plan.L.tmo_grav_plan_solve, C.c_void_p) if plan is not None else None
        rc = self.L.tmref_gravity_hydro_step(self.h, dt, cfl, gamma, workers, max_slices,
                                             solves_per_step if plan is not None else 0, fn,
                                             plan.h if plan is not None else None, grav_flags,
                                             C.byref(used), secs, err, 256)
        if rc != 0:
            raise RuntimeError(f"reference gravity+hydro step failed: {err.value.decode()}")
        return used.value, {"exchange_s": secs[0], "stage_s": secs[1], "gravity_s": secs[2],
                            "cfl_s": secs[3]}

    def hydro_step(self, dt, gamma=1.4, workers=1, lane_width=1, max_slices=8):
        tex, tst = C.c_double(0), C.c_double(0)
        err = C.create_string_buffer(256)
        rc = self.L.tmref_hydro_step(self.h, dt, gamma, workers, lane_width, max_slices,
                                     C.byref(tex), C.byref(tst), err, 256)
        if rc != 0:
            raise RuntimeError(f"reference hydro step failed: {err.value.decode()}")
        return tex.value, tst.value


def host_has_avx2_fma() -> bool:
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("flags"):
                    f = set(line.split(":", 1)[1].split())
                    return {"avx2", "fma", "bmi2"} <= f
    except OSError:
        pass
    return False


class Oracle(_Lib):
    """Our plain-C restatement (oracle/tm_oracle.c, gravity_*.c).

    fast=None picks liboracle_fast.so (the same sources, -O3 -march=x86-64-v3)
    on hosts with AVX2 + FMA, else the portable liboracle.so; both give the
    same bits (tests/test_gravity_amr.py)."""

    def __init__(self, fast=None):
        if fast is None:
            fast = host_has_avx2_fma() and os.path.exists(os.path.join(REF_DIR, "liboracle_fast.so"))
        super().__init__("liboracle_fast.so" if fast else "liboracle.so")
        self.fast = bool(fast)
        L = self.lib
        for f in ("tmo_minmod_scalar", "tmo_minmod_lane"):
            getattr(L, f).restype = C.c_double
            getattr(L, f).argtypes = [C.c_double, C.c_double]
        L.tmo_reconstruct_face.argtypes = [C.c_double] * 4 + [_dp]
        L.tmo_rusanov_euler.argtypes = [_dp, _dp, C.c_double, C.c_int, _dp]
        L.tmo_rusanov_scalar.restype = C.c_double
        L.tmo_rusanov_scalar.argtypes = [C.c_double] * 3
        L.tmo_stage_subgrid.argtypes = [_dp, C.c_int, C.c_int, C.c_int, _dp, _dp, _ip]
        L.tmo_stage_fused.argtypes = [_dp, _dp, C.c_size_t, C.c_size_t, C.c_size_t, C.c_int,
                                      C.c_int, C.c_int, C.POINTER(C.c_size_t), _ip]
        L.tmo_max_wavespeed.restype = C.c_double
        L.tmo_max_wavespeed.argtypes = [_dp, C.c_int, C.c_int, C.c_int, _dp]
        L.tmo_rk3_combine.restype = C.c_double
        L.tmo_rk3_combine.argtypes = [C.c_int, C.c_double, C.c_double]
        L.tmo_morton_encode.argtypes = [C.c_int, C.c_uint64, C.c_uint64, C.c_uint64, _u64p]
        L.tmo_morton_decode.argtypes = [C.c_int, C.c_uint64, _u64p]
        L.tmo_morton_dfs_rank.restype = C.c_uint64
        L.tmo_morton_dfs_rank.argtypes = [C.c_int, C.c_uint64]
        L.tmo_partition_leaves.argtypes = [_u64p, C.c_size_t, C.c_int, _ip]
        L.tmo_tree_create.restype = C.c_void_p
        L.tmo_tree_create.argtypes = [C.c_int, C.c_int, C.c_int, _ip, _ip, _u64p, C.c_size_t]
        L.tmo_tree_destroy.argtypes = [C.c_void_p]
        L.tmo_tree_leaves.restype = C.c_size_t
        L.tmo_tree_leaves.argtypes = [C.c_void_p, _u64p, C.c_size_t]
        L.tmo_tree_face_neighbor.argtypes = [C.c_void_p, C.c_uint64, C.c_int, C.c_int, _u64p, _ip]
        L.tmo_tree_plan.restype = C.c_size_t
        L.tmo_tree_plan.argtypes = [C.c_void_p, C.c_int, _i64p, C.c_size_t]
        L.tmo_fill_ghosts_sync.argtypes = [C.c_void_p, C.POINTER(_dp)]
        L.tmo_flag_refinement.argtypes = [C.c_void_p, _dp, C.c_double, C.c_double]
        L.tmo_reflux_apply.argtypes = [C.c_void_p, C.POINTER(_dp), C.POINTER(_dp), C.c_int, C.c_int, C.c_int, _dp, C.c_double, C.c_double]
        L.tmo_stage_subgrid_grav.argtypes = [_dp, C.c_int, C.c_int, C.c_int, _dp, _dp, _dp, _ip]
        _lp = C.POINTER(C.c_long)
        L.tmo_grav_amr_solve_ex.argtypes = [C.c_long, _ip, _dp, C.c_int, _dp, _dp, _lp]
        L.tmo_grav_amr_sparse.argtypes = [C.c_long, _ip, _dp, C.c_int, _dp, _dp, _lp]
        L.tmo_grav_plan_create.restype = C.c_void_p
        L.tmo_grav_plan_create.argtypes = [C.c_long, _ip, _ip]
        L.tmo_grav_plan_solve.argtypes = [C.c_void_p, _dp, C.c_int, _dp, _dp, _lp]
        L.tmo_grav_plan_destroy.argtypes = [C.c_void_p]
        L.tmo_grav_amr_direct.argtypes = [C.c_long, _ip, _dp, _dp, _dp]
        L.tmo_grav_am_correct.argtypes = [C.c_long, _dp, _dp, _dp, _dp, _dp]

    def grav_amr(self, leaves, mass, flags=0, direct=False, sparse=False):
        """AMR FMM specification (gravity_amr_oracle.c; sparse=True: the
        patch-sparse restatement gravity_amr_sparse.c, same bits, any depth).
        leaves: [n, 4] int (level, I, J, K) in canonical order; mass: [n, 512].
        Returns (phi[n*512], g[3, n*512], (W/X entries, U-cross entries))."""
        lv = np.ascontiguousarray(leaves, dtype=np.int32).reshape(-1, 4)
        m = np.ascontiguousarray(mass, dtype=np.float64).reshape(-1)
        n = lv.shape[0]
        assert m.size == n * 512
        phi, g = np.zeros(n * 512), np.zeros(3 * n * 512)
        cnt = (C.c_long * 2)()
        ip = lv.ctypes.data_as(_ip)
        if direct:
            r = self.lib.tmo_grav_amr_direct(n, ip, dptr(m), dptr(phi), dptr(g))
        elif sparse:
            r = self.lib.tmo_grav_amr_sparse(n, ip, dptr(m), flags, dptr(phi), dptr(g), cnt)
        else:
            r = self.lib.tmo_grav_amr_solve_ex(n, ip, dptr(m), flags, dptr(phi), dptr(g), cnt)
        if r != 0:
            raise ValueError(f"oracle AMR gravity failed ({r})")
        return phi, g.reshape(3, -1), (cnt[0], cnt[1])

    def grav_plan(self, leaves):
        """Patch-sparse solver with the topology work done once (like the GPU's
        GravityAMR): returns a GravPlan whose solve(mass, flags) gives the bits
        of grav_amr."""
        return GravPlan(self, leaves)

    def stage_fused(self, packed_in, count, edge=8, ghost=2, vars=5):
        S = edge + 2 * ghost
        ins = 8 + vars * S ** 3
        outs = vars * edge ** 3 + 6 * vars * edge ** 2 + 1
        out = np.zeros(count * outs)
        bad_slice = C.c_size_t(0)
        cell = (C.c_int * 3)()
        rc = self.lib.tmo_stage_fused(dptr(packed_in), dptr(out), ins, outs, count, edge, ghost,
                                      vars, C.byref(bad_slice), cell)
        return rc, out, (bad_slice.value, tuple(cell))

    def max_wavespeed(self, header, ghosted, edge=8, ghost=2, vars=5):
        return self.lib.tmo_max_wavespeed(dptr(header), edge, ghost, vars, dptr(ghosted))

    def tree(self, leaves, edge=8, ghost=2, vars=5, root_dims=(1, 1, 1), bc=(0, 0, 0)):
        return OracleTree(self, leaves, edge, ghost, vars, root_dims, bc)


class GravPlan:
    def __init__(self, o: "Oracle", leaves):
        self.L = o.lib
        self.lv = np.ascontiguousarray(leaves, dtype=np.int32).reshape(-1, 4)
        self.n = self.lv.shape[0]
        rc = C.c_int(0)
        self.h = self.L.tmo_grav_plan_create(self.n, self.lv.ctypes.data_as(_ip), C.byref(rc))
        if not self.h:
            raise ValueError(f"oracle gravity plan failed ({rc.value})")

    def solve(self, mass, flags=0):
        m = np.ascontiguousarray(mass, dtype=np.float64).reshape(-1)
        assert m.size == self.n * 512
        phi, g = np.zeros(self.n * 512), np.zeros(3 * self.n * 512)
        cnt = (C.c_long * 2)()
        r = self.L.tmo_grav_plan_solve(self.h, dptr(m), flags, dptr(phi), dptr(g), cnt)
        if r != 0:
            raise ValueError(f"oracle AMR gravity failed ({r})")
        return phi, g.reshape(3, -1), (cnt[0], cnt[1])

    def __del__(self):
        if getattr(self, "h", None):
            self.L.tmo_grav_plan_destroy(self.h)
            self.h = None


class OracleTree:
    def __init__(self, o: Oracle, leaves, edge, ghost, vars, root_dims, bc):
        self.L = o.lib
        self.edge, self.ghost, self.vars = edge, ghost, vars
        lv = np.ascontiguousarray(np.asarray(leaves, dtype=np.uint64))
        self.h = self.L.tmo_tree_create(edge, ghost, vars, (C.c_int * 3)(*root_dims),
                                        (C.c_int * 3)(*bc), u64ptr(lv), len(lv))

    def __del__(self):
        if getattr(self, "h", None):
            self.L.tmo_tree_destroy(self.h)
            self.h = None

    def leaves(self):
        n = self.L.tmo_tree_leaves(self.h, None, 0)
        out = np.zeros(n, dtype=np.uint64)
        self.L.tmo_tree_leaves(self.h, u64ptr(out), n)
        return out

    def face_neighbor(self, packed, axis, direction):
        ids = np.zeros(4, dtype=np.uint64)
        cnt = C.c_int(0)
        kind = self.L.tmo_tree_face_neighbor(self.h, packed, axis, direction, u64ptr(ids),
                                             C.byref(cnt))
        return kind, [int(x) for x in ids[: cnt.value]]

    def plan(self, axis):
        n = self.L.tmo_tree_plan(self.h, axis, None, 0)
        rows = np.zeros((n, 7), dtype=np.int64)
        self.L.tmo_tree_plan(self.h, axis, rows.ctypes.data_as(_i64p), n)
        return rows

    def fill_ghosts(self, grids):
        """grids: list of float64 arrays in canonical leaf order (modified in place)."""
        arr = (_dp * len(grids))(*[dptr(g) for g in grids])
        if self.L.tmo_fill_ghosts_sync(self.h, arr) != 0:
            raise RuntimeError("oracle ghost fill failed")

    def reflux(self, grids, faces, dx, dt, coef):
        """tmo_reflux_apply: grids (ghosted, canonical order, modified in place),
        faces: per leaf [6][V][E^2] stage face fluxes, dx: per-leaf cell size."""
        ga = (_dp * len(grids))(*[dptr(g) for g in grids])
        fa = (_dp * len(faces))(*[dptr(f) for f in faces])
        d = np.ascontiguousarray(dx, dtype=np.float64)
        if self.L.tmo_reflux_apply(self.h, ga, fa, self.edge, self.ghost, self.vars, dptr(d),
                                   float(dt), float(coef)) != 0:
            raise RuntimeError("oracle reflux failed")

    def flag(self, grid, theta, rho_floor=1e-10):
        return bool(self.L.tmo_flag_refinement(self.h, dptr(grid), theta, rho_floor))


def pack(level, ci, cj, ck) -> int:
    """NodeId::packed (reference octree.hpp:29-33)."""
    return (level << 60) | (ci << 40) | (cj << 20) | ck


def unpack(p: int):
    p = int(p)
    return p >> 60, (p >> 40) & 0xFFFFF, (p >> 20) & 0xFFFFF, p & 0xFFFFF


def leaf_centres(leaves):
    """Cell centres [n*512, 3] of leaves [n, 4] = (level, I, J, K), unit cube."""
    lv = np.asarray(leaves, dtype=np.int64).reshape(-1, 4)
    c = np.arange(512)
    loc = np.stack([c & 7, (c >> 3) & 7, c >> 6], 1)
    gl = lv[:, None, 1:] * 8 + loc[None]
    h = 1.0 / (8.0 * (2.0 ** lv[:, 0]))
    return ((gl + 0.5) * h[:, None, None]).reshape(-1, 3)


def random_forest_leaves(rng, base=1, max_level=3, frac=0.3):
    """Random (unbalanced) octree over the unit cube: uniform at `base`, then
    each leaf below max_level refined with probability frac, repeatedly.
    Returns [n, 4] (level, I, J, K) in canonical (Morton depth-first) order."""
    def rec(level, i, j, k, out):
        if level < base or (level < max_level and rng.random() < frac):
            for c in range(8):
                rec(level + 1, 2 * i + (c & 1), 2 * j + ((c >> 1) & 1), 2 * k + (c >> 2), out)
        else:
            out.append((level, i, j, k))
    out = []
    rec(0, 0, 0, 0, out)
    return np.array(out, dtype=np.int32)


def random_state(rng: np.random.Generator, edge=8, ghost=2, euler=True, gamma=1.4):
    """Reference test_hydro.cpp:21-43 state distribution (rho,p ~ U(0.2,2),
    velocities ~ U(-0.5,0.5)), drawn with numpy: identical buffers are fed to
    every implementation, so the RNG itself need not match libstdc++."""
    S = edge + 2 * ghost
    n = S ** 3
    if not euler:
        return rng.uniform(0.2, 2.0, n)
    rho = rng.uniform(0.2, 2.0, n)
    u, v, w = (rng.uniform(-0.5, 0.5, n) for _ in range(3))
    p = rng.uniform(0.2, 2.0, n)
    e = p / (gamma - 1.0) + 0.5 * rho * (u * u + v * v + w * w)
    return np.concatenate([rho, rho * u, rho * v, rho * w, e])
