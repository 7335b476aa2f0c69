"""torchrun helper (gloo, CPU): every rank builds the distributed-gravity
host plan for its own slot range; rank 0 checks the ranges tile the leaves and
that the per-rank M2L/L2L patch sets cover the whole cell tree."""
import os
import sys

import torch.distributed as tdist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2412_15518_b200 import amr, dist  # noqa: E402
from paper_2412_15518_b200.gravity import amr_plan_need, forest_leaf_array  # noqa: E402


def main():
    tdist.init_process_group("gloo")
    rank, world = tdist.get_rank(), tdist.get_world_size()
    f = amr.build_scenario(amr.Scenario.rotating_star, 2, 4)
    leaves = forest_leaf_array(f)
    owner = dist.partition(f, world)
    lo, hi = dist.local_range(owner, rank)
    mine = {"rank": rank, "lo": lo, "hi": hi, "need": amr_plan_need(leaves, lo, hi)}
    got = [None] * world
    tdist.all_gather_object(got, mine)
    if rank == 0:
        n = len(leaves)
        total = amr_plan_need(leaves, 0, n)  # one rank owns everything: every patch
        bounds = sorted((g["lo"], g["hi"]) for g in got)
        assert bounds[0][0] == 0 and bounds[-1][1] == n, bounds
        assert all(bounds[i][1] == bounds[i + 1][0] for i in range(world - 1)), bounds
        for g in got:
            assert g["need"][0] == 1, "every rank evaluates the root patch"
            assert all(a <= t for a, t in zip(g["need"], total))
        for l in range(len(total)):  # every patch is some rank's ancestor-or-self
            assert sum(g["need"][l] for g in got) >= total[l]
        print("GRAV_OK", world, n, total, [g["need"] for g in got])
    tdist.barrier()
    if rank != 0:
        print("GRAV_OK", rank)
    tdist.destroy_process_group()


if __name__ == "__main__":
    main()
