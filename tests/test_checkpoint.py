"""Checkpoint format: byte layout, round trip, error
behaviour, the multi-rank merge (gloo, world_size 2) on CPU; on the GPU the
determinism contract (same config + seed -> identical checkpoint bytes) and
save -> load -> save through the device arena."""
import os
import struct
import subprocess
import sys

import numpy as np
import pytest

from paper_2412_15518_b200 import amr, checkpoint

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _star(max_level=3):
    f = amr.build_scenario(amr.Scenario.rotating_star, 2, max_level)
    return f, f.scenario_state(amr.Scenario.rotating_star)


def test_layout_little_endian():
    keys = np.array([amr.pack(1, 0, 0, 0), amr.pack(1, 1, 0, 0)], dtype=np.uint64)
    payload = np.arange(2 * 5 * 512, dtype=np.float64).reshape(2, 5, 512)
    buf = checkpoint.encode(keys, payload, time=1.5, step=7)
    assert len(buf) == checkpoint.HEADER_BYTES + 2 * (8 + 5 * 512 * 8)
    assert buf[:4] == b"TMCK" and buf[4] == 2 and buf[5] == 0
    assert struct.unpack_from("<HH", buf, 6) == (5, 8) and buf[10] == 0 and buf[11:16] == bytes(5)
    assert struct.unpack_from("<dQQ", buf, 16) == (1.5, 7, 2)
    off = checkpoint.HEADER_BYTES
    assert struct.unpack_from("<Q", buf, off)[0] == int(keys[0])
    assert struct.unpack_from("<3d", buf, off + 8) == (0.0, 1.0, 2.0)
    rec = 8 + 5 * 512 * 8
    assert struct.unpack_from("<Q", buf, off + rec)[0] == int(keys[1])
    assert struct.unpack_from("<d", buf, off + rec + 8)[0] == 2560.0


def test_round_trip_bitwise():
    f, st = _star()
    st = st.copy()
    st[0, 0, 0] = -0.0
    st[1, 4, 3] = np.nextafter(1.0, 2.0)
    buf = checkpoint.encode(f.leaves(), st, time=0.125, step=2)
    head, keys, payload = checkpoint.decode(buf)
    assert head == {"version": 2, "flags": 0, "vars": 5, "edge": 8, "ghost": 0, "time": 0.125, "step": 2,
                    "records": f.leaf_count()}
    assert (keys == f.leaves()).all()
    assert payload.tobytes() == st.tobytes()
    assert checkpoint.encode(keys, payload, 0.125, 2) == buf


def test_scalar_mode_and_empty():
    keys = np.array([amr.pack(0, 0, 0, 0)], dtype=np.uint64)
    buf = checkpoint.encode(keys, np.ones((1, 1, 512)))
    head, _, payload = checkpoint.decode(buf)
    assert head["vars"] == 1 and payload.shape == (1, 1, 512)
    head, keys, payload = checkpoint.decode(checkpoint.encode([], np.zeros((0, 5, 512))))
    assert head["records"] == 0 and keys.size == 0 and payload.shape == (0, 5, 512)


def test_rejects_corrupt_files():
    f, st = _star()
    buf = checkpoint.encode(f.leaves(), st)
    with pytest.raises(checkpoint.CheckpointError, match="magic"):
        checkpoint.decode(b"XXXX" + buf[4:])
    with pytest.raises(checkpoint.CheckpointError, match="version"):
        checkpoint.decode(buf[:4] + b"\x07" + buf[5:])
    with pytest.raises(checkpoint.CheckpointError, match="record bytes"):
        checkpoint.decode(buf[:-8])
    with pytest.raises(checkpoint.CheckpointError, match="header"):
        checkpoint.decode(buf[:10])
    with pytest.raises(checkpoint.CheckpointError, match="does not match"):
        checkpoint.encode(f.leaves()[:-1], st)


def test_merge_canonical_order_and_errors():
    f, st = _star()
    lv = f.leaves()
    n = len(lv)
    # ranks contribute out of order; the merge restores the canonical order
    parts = [(lv[n // 2:], st[n // 2:]), (lv[: n // 2], st[: n // 2])]
    order, out = checkpoint.merge(lv, parts)
    assert out.tobytes() == st.tobytes()
    with pytest.raises(checkpoint.CheckpointError, match="missing"):
        checkpoint.merge(lv, parts[:1])
    with pytest.raises(checkpoint.CheckpointError, match="twice"):
        checkpoint.merge(lv, parts + [(lv[:1], st[:1])])


def test_save_without_device_state(tmp_path):
    f, st = _star()
    p = tmp_path / "c.tmck"
    buf = checkpoint.save(str(p), f, time=0.5, step=1, state=st)
    assert p.read_bytes() == buf == checkpoint.encode(f.leaves(), st, 0.5, 1)


def test_gloo_world2_merged_checkpoint_equals_single_process(tmp_path):
    env = dict(os.environ, GLOO_SOCKET_IFNAME="lo", CKPT_PATH=str(tmp_path / "ranged.tmck"))
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        "--nproc-per-node=2", "--master-addr", "127.0.0.1", "--master-port",
                        "29567", os.path.join(ROOT, "tests", "gloo_checkpoint.py")],
                       capture_output=True, text=True, timeout=300, env=env)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert r.stdout.count("CKPT_OK") == 2, r.stdout[-2000:]


@pytest.mark.gpu
def test_checkpoint_determinism_and_reload(tmp_path):
    """identical config + seed run twice -> identical checkpoint
    bytes; a saved state loaded into a fresh forest saves to the same bytes.
    (Resuming from these interior records is not bitwise — the step carries
    ghost-layer values across exchanges — which is what the RESUMABLE format is
    for: test_resumable_checkpoint_continues_bitwise.)"""
    from paper_2412_15518_b200.driver import HydroDriver

    files = []
    for run in range(2):
        f = amr.build_scenario(amr.Scenario.rotating_star, 2, 4)
        f.alloc()
        f.set_interior(f.scenario_state(amr.Scenario.rotating_star))
        drv = HydroDriver(f)
        t = 0.0
        for _ in range(2):
            t += drv.step()
        p = tmp_path / f"run{run}.tmck"
        checkpoint.save(str(p), f, time=t, step=2)
        files.append(p.read_bytes())
    assert files[0] == files[1]
    head, keys, payload = checkpoint.decode(files[0])
    assert head["records"] == f.leaf_count() and (keys == f.leaves()).all()
    assert payload.tobytes() == f.get_interior().tobytes()
    g = amr.build_scenario(amr.Scenario.rotating_star, 2, 4)
    g.alloc()
    head = checkpoint.load(str(tmp_path / "run0.tmck"), g)
    assert head["step"] == 2 and head["time"] == t
    assert checkpoint.save(None, g, time=head["time"], step=2) == files[0]


def test_version1_files_still_load():
    """A version-1 file (no ghost byte) decodes like a version-2 interior file."""
    f = amr.build_scenario(amr.Scenario.rotating_star, 1, 2)
    st = f.scenario_state(amr.Scenario.rotating_star)
    buf = bytearray(checkpoint.encode(f.leaves(), st, 0.5, 3))
    buf[4] = 1  # version 1
    buf[10] = 0  # its reserved byte where version 2 keeps the ghost width
    head, keys, payload = checkpoint.decode(bytes(buf))
    assert head["version"] == 1 and head["ghost"] == 0 and payload.tobytes() == st.tobytes()


def test_resumable_encode_roundtrip():
    blocks = np.random.default_rng(3).normal(size=(3, 2, 5, 12 ** 3))
    keys = np.array([1, 2, 3], dtype=np.uint64)
    buf = checkpoint.encode(keys, blocks, 0.25, 9, ghost=2, flags=checkpoint.RESUMABLE)
    assert len(buf) == checkpoint.HEADER_BYTES + 3 * (8 + 2 * 5 * 12 ** 3 * 8)
    head, k, p = checkpoint.decode(buf)
    assert head["flags"] == checkpoint.RESUMABLE and head["ghost"] == 2
    assert (k == keys).all() and p.tobytes() == blocks.tobytes()
    with pytest.raises(checkpoint.CheckpointError, match="ghost"):
        checkpoint.encode(keys, blocks, flags=checkpoint.RESUMABLE)


def test_merge_of_no_records():
    order, out = checkpoint.merge([], [([], np.zeros((0, 5, 512)))])
    assert len(order) == 0
    with pytest.raises(checkpoint.CheckpointError, match="missing"):
        checkpoint.merge([1, 2], [([], np.zeros((0, 5, 512)))])


@pytest.mark.gpu
@pytest.mark.parametrize("gravity", [False, True])
def test_resumable_checkpoint_continues_bitwise(tmp_path, gravity):
    """save(resumable) -> load into a fresh forest -> step == stepping on
    uninterrupted, bit for bit (SPEC.md:425's "bitwise equivalence" use)."""
    from paper_2412_15518_b200.driver import GravityHydroDriver, HydroDriver

    Drv = GravityHydroDriver if gravity else HydroDriver

    def fresh():
        f = amr.build_scenario(amr.Scenario.rotating_star, 2, 4)
        f.alloc()
        return f

    f = fresh()
    f.set_interior(f.scenario_state(amr.Scenario.rotating_star))
    drv = Drv(f)
    for _ in range(3):
        drv.step()
    p = tmp_path / "resume.tmck"
    checkpoint.save(str(p), f, time=0.0, step=3, resumable=True)
    dts = [drv.step() for _ in range(2)]
    want = f.get_interior()
    g = fresh()
    head = checkpoint.load(str(p), g)
    assert head["flags"] & checkpoint.RESUMABLE and head["step"] == 3
    d2 = Drv(g)
    dts2 = [d2.step() for _ in range(2)]
    assert dts2 == dts
    assert g.get_interior().tobytes() == want.tobytes()
