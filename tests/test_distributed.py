"""Leaf-to-GPU distribution: partition + halo plan consistency (CPU, incl. a
world_size-2 gloo run), and the partitioned multi-GPU step vs the 1-GPU step
(bitwise) when two GPUs are present."""
import os
import subprocess
import sys

import numpy as np
import pytest

from paper_2412_15518_b200 import amr, dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _pair_consistent(f, owner, world):
    """Rank q's slabs to r are, in order, rank r's expected slabs from q."""
    man = [f.halo_manifest(owner, r, world) for r in range(world)]
    for r in range(world):
        for q in range(world):
            if q == r:
                continue
            sent = man[q][(man[q][:, 0] == 0) & (man[q][:, 1] == r)][:, 2:]
            recv = man[r][(man[r][:, 0] == 1) & (man[r][:, 1] == q)][:, 2:]
            assert sent.shape == recv.shape
            assert (sent == recv).all()
    return man


@pytest.mark.parametrize("world", [2, 3, 4, 8])
def test_halo_plan_pairwise_consistent(world):
    f = amr.build_scenario(amr.Scenario.rotating_star, 2, 4)
    owner = dist.partition(f, world)
    assert owner == amr.partition_leaves([512] * f.leaf_count(), world)
    man = _pair_consistent(f, owner, world)
    # every cross-rank fill of the reference plan appears exactly once
    lv = [int(p) for p in f.leaves()]
    idx = {p: i for i, p in enumerate(lv)}
    cross = 0
    for axis in range(3):
        for row in f.plan(axis):
            dst, src, kind = int(row[0]), int(row[1]), int(row[2])
            if kind != 3 and owner[idx[dst]] != owner[idx[src]]:
                cross += 1
    assert sum(int((m[:, 0] == 0).sum()) for m in man) == cross


def test_local_ranges_contiguous():
    f = amr.build_scenario(amr.Scenario.sod, 2, 4, bc=(0, 1, 1))
    owner = dist.partition(f, 4)
    covered = 0
    for r in range(4):
        lo, hi = dist.local_range(owner, r)
        assert all(o == r for o in owner[lo:hi])
        covered += hi - lo
    assert covered == f.leaf_count()


def test_gloo_world2_halo_manifests_agree():
    """Two processes (torch.distributed gloo, world_size 2) build their own
    halo plans and exchange them: rank q's sends to r == r's expected receipts."""
    env = dict(os.environ, GLOO_SOCKET_IFNAME="lo")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        "--nproc-per-node=2", "--master-addr", "127.0.0.1", "--master-port",
                        "29563", os.path.join(ROOT, "tests", "gloo_halo.py")],
                       capture_output=True, text=True, timeout=300, env=env)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert r.stdout.count("HALO_OK") == 2, r.stdout[-2000:]


def test_gloo_world2_gravity_partition():
    """Two processes (gloo, world_size 2): the distributed FMM's slot ranges tile
    the leaves and the per-rank M2L/L2L patch sets cover the cell tree."""
    env = dict(os.environ, GLOO_SOCKET_IFNAME="lo")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        "--nproc-per-node=2", "--master-addr", "127.0.0.1", "--master-port",
                        "29564", os.path.join(ROOT, "tests", "gloo_gravity.py")],
                       capture_output=True, text=True, timeout=300, env=env)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert r.stdout.count("GRAV_OK") == 2, r.stdout[-2000:]


@pytest.mark.gpu
def test_partitioned_step_bitwise_equals_single_gpu():
    import torch

    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs (gpurun --gpus 2)")
    script = os.path.join(ROOT, "tests", "mgpu_step.py")
    out = os.path.join(ROOT, "gpurun_out", "mgpu_step.npz") if os.path.isdir(
        os.path.join(ROOT, "gpurun_out")) else "/tmp/mgpu_step.npz"
    n = min(torch.cuda.device_count(), 4)
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        f"--nproc-per-node={n}", "--master-addr", "127.0.0.1", "--master-port",
                        "29531", script, out], capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "BITWISE_OK" in r.stdout, r.stdout[-3000:]


@pytest.mark.gpu
def test_partitioned_gravity_hydro_step_bitwise_equals_single_gpu():
    """Distributed FMM (mass all-gather, owned-subtree M2L/L2L/L2P, all-gathered
    AM sums) + partitioned hydro == one GPU, bitwise (state and gravity field)."""
    import torch

    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs (gpurun --gpus 2)")
    script = os.path.join(ROOT, "tests", "mgpu_step.py")
    n = min(torch.cuda.device_count(), 4)
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        f"--nproc-per-node={n}", "--master-addr", "127.0.0.1", "--master-port",
                        "29532", script, "--gravity"], capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "BITWISE_OK" in r.stdout, r.stdout[-3000:]


@pytest.mark.gpu
@pytest.mark.parametrize("gravity", [False, True])
def test_peer_halo_step_bitwise_equals_single_gpu(gravity):
    """Ghost slabs stored straight into the peers' buffers (CUDA IPC, flag-word
    sync) instead of NCCL send/recv: same bits as one GPU."""
    import torch

    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs (gpurun --gpus 2)")
    script = os.path.join(ROOT, "tests", "mgpu_step.py")
    n = min(torch.cuda.device_count(), 4)
    extra = ["--peer"] + (["--gravity"] if gravity else [])
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        f"--nproc-per-node={n}", "--master-addr", "127.0.0.1", "--master-port",
                        str(29533 + int(gravity)), script] + extra, capture_output=True, text=True,
                       timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "BITWISE_OK" in r.stdout, r.stdout[-3000:]


@pytest.mark.gpu
@pytest.mark.parametrize("extra", [["--regrid"], ["--regrid", "--gravity", "--peer"], ["--reflux"],
                                   ["--reflux", "--gravity", "--peer", "--regrid"]])
def test_distributed_regrid_reflux_bitwise_equals_single_gpu(extra):
    """Collective regrid of a distributed forest (dist.regrid: refine with 2:1
    cascades and coarsen with the data carried along, re-partition, blocks moved
    to their new owners; peer exchanges rebuilt) and two more steps, and/or
    reflux with the fine face blocks exchanged across GPUs after every stage ==
    the same on one GPU, bitwise (state, gravity field, checkpoint bytes)."""
    import torch

    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs (gpurun --gpus 2)")
    script = os.path.join(ROOT, "tests", "mgpu_step.py")
    n = min(torch.cuda.device_count(), 4)
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        f"--nproc-per-node={n}", "--master-addr", "127.0.0.1", "--master-port",
                        str(29541 + len(extra) + 7 * ("--reflux" in extra)), script] + extra,
                       capture_output=True, text=True,
                       timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "BITWISE_OK" in r.stdout, r.stdout[-3000:]


@pytest.mark.gpu
def test_peer_wait_is_bounded_when_a_peer_stops():
    """A rank whose peer stops stepping fails its next peer-memory step after
    TMGPU_PEER_TIMEOUT_S instead of hanging (tests/mgpu_peer_timeout.py)."""
    import torch

    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs (gpurun --gpus 2)")
    script = os.path.join(ROOT, "tests", "mgpu_peer_timeout.py")
    env = dict(os.environ, TMGPU_PEER_TIMEOUT_S="2", CUDA_VISIBLE_DEVICES="0,1")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
                        "--master-addr", "127.0.0.1", "--master-port", "29539", script],
                       capture_output=True, text=True, timeout=180, env=env)
    assert "PEER_TIMEOUT_OK" in r.stdout, r.stdout[-3000:] + r.stderr[-3000:]
    elapsed = float(r.stdout.split("PEER_TIMEOUT_OK")[1].split()[0])
    assert elapsed < 15.0, r.stdout[-2000:]

