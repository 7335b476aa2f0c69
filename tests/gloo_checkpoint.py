"""torchrun helper (gloo, CPU): every rank contributes the records of its
partition_leaves range of the 4-level star's initial state; rank 0's merged
checkpoint must equal the one-process file byte for byte."""
import os
import sys

import numpy as np
import torch.distributed as tdist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2412_15518_b200 import amr, checkpoint, dist  # noqa: E402

tdist.init_process_group("gloo")
rank, world = tdist.get_rank(), tdist.get_world_size()
f = amr.build_scenario(amr.Scenario.rotating_star, 2, 4)
state = f.scenario_state(amr.Scenario.rotating_star)
owner = np.asarray(dist.partition(f, world))
mine = owner == rank
buf = checkpoint.save(None, f, time=0.25, step=3, state=state[mine], keys=f.leaves()[mine])
single = checkpoint.encode(f.leaves(), state, time=0.25, step=3)
ok = (buf == single) if rank == 0 else (buf is None)
# with a path: every rank writes its own byte range, nothing is gathered
path = os.environ.get("CKPT_PATH", "/tmp/gloo_ckpt.tmck")
ret = checkpoint.save(path, f, time=0.25, step=3, state=state[mine], keys=f.leaves()[mine])
tdist.barrier()
with open(path, "rb") as fh:
    ok = ok and ret is None and fh.read() == single
print("CKPT_OK" if ok else "CKPT_MISMATCH", rank)
tdist.destroy_process_group()
