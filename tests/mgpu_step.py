"""torchrun helper for test_distributed: partitioned steps on N GPUs vs one GPU.

Each rank owns a contiguous range of canonical leaves; after 3 SSP-RK3 steps
(hydro, or gravity+hydro with `--gravity`: distributed FMM solve + hydro) the
ranks gather their interiors (and the last gravity field) on rank 0, which
reruns the same steps on one GPU and compares bitwise (state, gravity field,
and the merged checkpoint file's bytes)."""
import os
import sys

import numpy as np
import torch
import torch.distributed as tdist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2412_15518_b200 import amr, checkpoint, dist  # noqa: E402
from paper_2412_15518_b200.driver import GravityHydroDriver, HydroDriver  # noqa: E402


def regrid_lists(f):
    """A deterministic refine + coarsen request every rank computes alike: three
    level-3 leaves refined, then up to two parents of 8 leaf children (not among
    them) coarsened where the 2:1 rule allows (tried on a topology copy)."""
    lv = [int(p) for p in f.leaves()]
    refine = [p for p in lv if amr.unpack(p)[0] == 3][::97][:3]
    g = dist.replay_topology(f, lv)
    for p in refine:
        g.refine(p)
    have = set(int(p) for p in g.leaves())
    coarsen = []
    for p in sorted(have):
        lvl, i, j, k = amr.unpack(p)
        if lvl < 2:
            continue
        par = amr.pack(lvl - 1, i >> 1, j >> 1, k >> 1)
        kids = [amr.pack(lvl, 2 * (i >> 1) + (b & 1), 2 * (j >> 1) + ((b >> 1) & 1), 2 * (k >> 1) + (b >> 2))
                for b in range(8)]
        if par in coarsen or not all(c in have for c in kids):
            continue
        try:
            g.coarsen(par)
        except amr.AmrError:
            continue
        have = set(int(q) for q in g.leaves())
        coarsen.append(par)
        if len(coarsen) == 2:
            break
    return refine, coarsen


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    tdist.init_process_group("nccl", device_id=torch.device("cuda", local))
    gravity = "--gravity" in sys.argv
    peer = "--peer" in sys.argv
    regrid = "--regrid" in sys.argv
    reflux = "--reflux" in sys.argv
    args = [a for a in sys.argv[1:] if a not in ("--gravity", "--peer", "--regrid", "--reflux")]
    Drv = GravityHydroDriver if gravity else HydroDriver
    kind, lo, hi = amr.Scenario.rotating_star, 2, 4
    f = amr.build_scenario(kind, lo, hi)
    state = f.scenario_state(kind)
    owner = dist.partition(f, world)
    comm = dist.Comm.from_torch()
    f.distribute(comm, owner)
    f.alloc()
    if peer:
        f.set_peer(True)
    a, b = dist.local_range(owner, rank)
    f.set_interior(np.ascontiguousarray(state[a:b]))
    drv = Drv(f, reflux=reflux)
    dts = [drv.step() for _ in range(3)]
    if regrid:  # collective regrid + re-partition, then more steps
        rl, cl = regrid_lists(f)
        drv.regrid(rl, cl)
        dts += [drv.step() for _ in range(2)]
        owner = f._owner
    ckpt = checkpoint.save(None, f, time=sum(dts), step=3)  # collective: rank 0 merges
    # collective, nothing gathered: every rank writes its own byte range
    cpath = os.path.join(os.environ.get("TMPDIR", "/tmp"), f"mgpu_ckpt_{os.getpid() if rank == 0 else 0}.tmck")
    cpath = [cpath]
    tdist.broadcast_object_list(cpath, src=0)
    assert checkpoint.save(cpath[0], f, time=sum(dts), step=3) is None
    mine = torch.from_numpy(f.get_interior()).cuda()
    sizes = [dist.local_range(owner, r)[1] - dist.local_range(owner, r)[0] for r in range(world)]
    gathered = [torch.zeros((s, 5, 512), dtype=torch.float64, device="cuda") for s in sizes]
    tdist.all_gather(gathered, mine)
    if gravity:
        gl = [torch.zeros((3, s * 512), dtype=torch.float64, device="cuda") for s in sizes]
        tdist.all_gather(gl, drv.g.view(3, -1).contiguous())
    if rank == 0:
        multi = torch.cat(gathered).cpu().numpy()
        g = amr.build_scenario(kind, lo, hi)
        g.alloc()
        g.set_interior(state)
        d1 = Drv(g, reflux=reflux)
        dts1 = [d1.step() for _ in range(3)]
        if regrid:
            d1.regrid(rl, cl)
            dts1 += [d1.step() for _ in range(2)]
            assert np.array_equal(g.leaves(), f.leaves())
        single = g.get_interior()
        assert dts == dts1, (dts, dts1)
        assert ckpt == checkpoint.encode(g.leaves(), single, sum(dts1), 3), "checkpoint differs"
        with open(cpath[0], "rb") as fh:
            assert fh.read() == ckpt, "ranged checkpoint write differs"
        os.remove(cpath[0])
        if gravity:
            gm = torch.cat(gl, dim=1).cpu().numpy()
            gs = d1.g.view(3, -1).cpu().numpy()
            assert gm.tobytes() == gs.tobytes(), "gravity field differs"
            d1.close()
        if multi.tobytes() == single.tobytes():
            print("BITWISE_OK", world, f.leaf_count(), dts)
        else:
            bad = np.nonzero((multi != single).any(axis=(1, 2)))[0]
            print("MISMATCH leaves", bad[:20], len(bad))
        if args:
            np.savez(args[0], multi=multi, single=single)
    drv.release_peers()  # collective peer-exchange teardown (also closes the gravity solver)
    tdist.barrier()
    tdist.destroy_process_group()


if __name__ == "__main__":
    main()
