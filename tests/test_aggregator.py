"""Kernel-aggregation executor: the reference's own aggregation tests
(proj/tests/test_aggregator.cpp) replayed against the CUDA-stream executor.

Pool bookkeeping is host-only (CPU tests); region launches run on the B200.
"""
import threading

import numpy as np
import pytest

from oracle import oracle as O
from paper_2412_15518_b200 import aggregator as A
from paper_2412_15518_b200 import hydro as H


# ------------------------------------------------------------------ pool (CPU)
def test_acquire_round_robin_on_idle_pool():
    """test_aggregator.cpp:49-56."""
    pool = A.ExecutorPool(4)
    held = [pool.acquire() for _ in range(4)]
    assert [h.index() for h in held] == [0, 1, 2, 3]


def test_acquire_least_loaded():
    """test_aggregator.cpp:58-68: counters [2,0,1,1] -> 1."""
    pool = A.ExecutorPool(4)
    held = [pool.acquire_at(0), pool.acquire_at(0), pool.acquire_at(2), pool.acquire_at(3)]
    assert pool.acquire().index() == 1
    del held


def test_concurrent_acquires_balance():
    """test_aggregator.cpp:70-89: 128 concurrent acquires on P=8."""
    pool = A.ExecutorPool(8)
    held, mu = [], threading.Lock()

    def work():
        for _ in range(16):
            lease = pool.acquire()
            with mu:
                held.append(lease)

    ts = [threading.Thread(target=work) for _ in range(8)]
    [t.start() for t in ts]
    [t.join() for t in ts]
    assert len(held) == 128
    assert all(pool.in_flight(e) == 16 for e in range(8))
    for h in held:
        h.reset()
    assert all(pool.in_flight(e) == 0 for e in range(8))


def test_pool_contract_errors():
    with pytest.raises(A.AggError):
        A.ExecutorPool(0)
    reg = A.KernelRegistry()
    spec = H.make_stage_kernel(H.StageGeom(vars=5), 1, 7)
    reg.add(spec)
    assert reg.at(7) is spec
    with pytest.raises(A.AggError):
        reg.add(spec)
    with pytest.raises(A.AggError):
        reg.at(8)


# ------------------------------------------------------------------ regions (GPU)
def affine(n):
    """The reference tests' toy kernel y = 2x + 1 (test_aggregator.cpp:17-29) as a
    registered device kernel; it lives in tools/probes/libtmprobe.so, not in the
    product library."""
    import ctypes as C
    import os
    import sys

    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                    "tools", "probes"))
    import probe

    fn = C.cast(probe.load().tmprobe_affine_launch, C.c_void_p).value
    return A.DeviceKernel(fn, n, n)


class Rig:
    def __init__(self):
        self.execs = A.ExecutorPool(4)
        self.counters = A.AggCounters()

    def pin_all_busy(self):
        return [self.execs.acquire() for _ in range(self.execs.size())]


@pytest.mark.gpu
def test_full_batch_launches_once():
    """test_aggregator.cpp:91-107."""
    rig = Rig()
    busy = rig.pin_all_busy()
    region = A.AggregationRegion(rig.execs, affine(4), 4, 16, rig.counters)
    futs = [region.submit_slice([1, 2, 3, 4]) for _ in range(4)]
    outs = A.when_all(futs)
    assert rig.counters.launches == 1 and rig.counters.fused_slices == 4
    for out in outs:
        assert out[0] == 3.0 and out[3] == 9.0
    del busy


@pytest.mark.gpu
def test_five_submits_busy_launch_4_plus_1():
    """test_aggregator.cpp:109-122."""
    rig = Rig()
    busy = rig.pin_all_busy()
    region = A.AggregationRegion(rig.execs, affine(2), 4, 16, rig.counters)
    futs = [region.submit_slice([0, 0]) for _ in range(5)]
    assert rig.counters.launches == 1
    region.flush()
    assert rig.counters.launches == 2 and rig.counters.solo_launches == 1
    A.when_all(futs)
    del busy


@pytest.mark.gpu
def test_idle_executor_launches_immediately():
    """test_aggregator.cpp:124-134."""
    rig = Rig()
    region = A.AggregationRegion(rig.execs, affine(2), 4, 16, rig.counters)
    f = region.submit_slice([5, 6])
    assert rig.counters.launches == 1 and rig.counters.fused_slices == 1
    assert f.get()[0] == 11.0


@pytest.mark.gpu
def test_flush_empty_and_idempotent():
    """test_aggregator.cpp:136-159."""
    rig = Rig()
    busy = rig.pin_all_busy()
    region = A.AggregationRegion(rig.execs, affine(2), 4, 16, rig.counters)
    region.flush()
    region.flush()
    assert rig.counters.launches == 0
    r2 = A.AggregationRegion(rig.execs, affine(2), 8, 16, rig.counters)
    futs = [r2.submit_slice([0, 0]) for _ in range(3)]
    r2.flush()
    r2.flush()
    assert rig.counters.launches == 1 and rig.counters.fused_slices == 3
    A.when_all(futs)
    del busy


@pytest.mark.gpu
def test_contract_errors():
    """test_aggregator.cpp:161-170."""
    rig = Rig()
    region = A.AggregationRegion(rig.execs, affine(2), 4, 16, rig.counters)
    with pytest.raises(A.AggError):
        region.submit_slice([1, 2, 3])
    region.flush()
    with pytest.raises(A.AggError):
        region.submit_slice([1, 2])
    with pytest.raises(A.AggError):
        A.AggregationRegion(rig.execs, affine(2), 0, 16)


@pytest.mark.gpu
@pytest.mark.parametrize("max_slices", [1, 3, 8, 100])
def test_fused_equals_solo_bitwise(max_slices):
    """test_aggregator.cpp:172-207 + launch-count bounds."""
    rng = np.random.default_rng(2024)
    inputs = rng.uniform(-100, 100, (100, 8))
    solo = 2.0 * inputs + 1.0
    rig = Rig()
    busy = rig.pin_all_busy()
    region = A.AggregationRegion(rig.execs, affine(8), max_slices, 100, rig.counters)
    futs = [region.submit_slice(s) for s in inputs]
    region.flush()
    for f, want in zip(futs, solo):
        assert f.get().tobytes() == want.tobytes()
    assert -(-100 // max_slices) <= rig.counters.launches <= 100
    del busy


@pytest.mark.gpu
def test_monotone_batching():
    """test_aggregator.cpp:209-223."""
    rig = Rig()
    busy = rig.pin_all_busy()
    region = A.AggregationRegion(rig.execs, affine(2), 4, 28, rig.counters)
    futs = [region.submit_slice([0, 0]) for _ in range(28)]
    assert rig.counters.launches == 7
    region.flush()
    assert rig.counters.launches == 7
    A.when_all(futs)
    del busy


@pytest.mark.gpu
def test_no_lost_slices_under_concurrency():
    """test_aggregator.cpp:225-247: 3 submitter threads x 200."""
    rig = Rig()
    region = A.AggregationRegion(rig.execs, affine(4), 8, 600, rig.counters)
    futs, mu = [], threading.Lock()

    def work():
        for _ in range(200):
            f = region.submit_slice([1, 2, 3, 4])
            with mu:
                futs.append(f)

    ts = [threading.Thread(target=work) for _ in range(3)]
    [t.start() for t in ts]
    [t.join() for t in ts]
    region.flush()
    outs = A.when_all(futs)
    assert len(outs) == 600 and rig.counters.fused_slices == 600
    assert all(o[1] == 5.0 for o in outs)


@pytest.mark.gpu
def test_in_flight_returns_to_zero():
    """test_aggregator.cpp:249-262."""
    rig = Rig()
    region = A.AggregationRegion(rig.execs, affine(2), 2, 32, rig.counters)
    futs = [region.submit_slice([0, 0]) for _ in range(32)]
    region.flush()
    A.when_all(futs)
    region.close()
    assert all(rig.execs.in_flight(e) == 0 for e in range(4))


@pytest.mark.gpu
@pytest.mark.parametrize("max_slices", [1, 8])
def test_stage_region_matches_reference(max_slices):
    """The hydro stage through the GPU region == the reference stage bitwise,
    for any batching (aggregation transparency)."""
    rng = np.random.default_rng(77)
    g = H.StageGeom(vars=5)
    n = 24
    slices = []
    for s in range(n):
        x = np.zeros(g.in_slice())
        dx = (1 / 64) * 2.0 ** -(s % 3)
        H.encode_header(H.StageParams(H.Mode.euler, dx, 0.2 * dx), x)
        x[8:] = O.random_state(rng)
        slices.append(x)
    rig = Rig()
    region = A.AggregationRegion(rig.execs, g, max_slices, n, rig.counters)
    futs = [region.submit_slice(x) for x in slices]
    region.flush()
    checker = O.Ref() if O.ref_available() else O.Oracle()
    rc, ref, _ = checker.stage_fused(np.concatenate(slices), n)
    assert rc == 0
    for s, f in enumerate(futs):
        assert f.get().tobytes() == ref[s * g.out_slice():(s + 1) * g.out_slice()].tobytes()


@pytest.mark.gpu
def test_stage_region_error_fails_whole_batch():
    """aggregator.cpp:164-167: an error fails every slice of the batch."""
    rng = np.random.default_rng(3)
    g = H.StageGeom(vars=5)
    rig = Rig()
    busy = rig.pin_all_busy()
    region = A.AggregationRegion(rig.execs, g, 4, 8, rig.counters)
    futs = []
    for s in range(4):
        x = np.zeros(g.in_slice())
        H.encode_header(H.StageParams(H.Mode.euler, 0.01, 0.001), x)
        x[8:] = O.random_state(rng)
        if s == 2:
            x[8 + 5 * 144 + 5 * 12 + 5] = np.nan
        futs.append(region.submit_slice(x))
    for f in futs:
        with pytest.raises(H.SolverError):
            f.get()
    del busy
