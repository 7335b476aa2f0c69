"""torchrun helper (gloo, CPU): every rank builds its halo plan for the
partitioned 4-level star and checks it against its peers' plans."""
import os
import sys

import numpy as np
import torch.distributed as tdist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2412_15518_b200 import amr, dist  # noqa: E402

tdist.init_process_group("gloo")
rank, world = tdist.get_rank(), tdist.get_world_size()
f = amr.build_scenario(amr.Scenario.rotating_star, 2, 4)
owner = dist.partition(f, world)
man = f.halo_manifest(owner, rank, world)
everything = [None] * world
tdist.all_gather_object(everything, man.tolist())
ok = len(man) > 0
for q in range(world):
    if q == rank:
        continue
    theirs = np.array(everything[q], dtype=np.int64).reshape(-1, 7)
    sent = theirs[(theirs[:, 0] == 0) & (theirs[:, 1] == rank)][:, 2:]
    recv = man[(man[:, 0] == 1) & (man[:, 1] == q)][:, 2:]
    ok &= sent.shape == recv.shape and bool((sent == recv).all())
print("HALO_OK" if ok else "HALO_MISMATCH", rank, len(man))
tdist.destroy_process_group()
