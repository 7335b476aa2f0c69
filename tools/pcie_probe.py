"""Host<->device copy throughput per rank with every rank copying at once
(torchrun --nproc-per-node N tools/pcie_probe.py MB): the floor under the
bench's e2e number (H2D of the step input and D2H of its result, concurrent)."""
import os
import sys

import torch
import torch.distributed as dist

mb = float(sys.argv[1]) if len(sys.argv) > 1 else 30.0
rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
local = int(os.environ.get("LOCAL_RANK", 0))
torch.cuda.set_device(local)
if world > 1:
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
n = int(mb * 2**20 / 8)
hi = torch.empty(n, dtype=torch.float64).pin_memory()
ho = torch.empty(n, dtype=torch.float64).pin_memory()
d1, d2 = torch.empty(n, dtype=torch.float64, device="cuda"), torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
res = {}
for mode in ("h2d", "d2h", "both"):
    for it in range(2):
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        s1.wait_stream(torch.cuda.current_stream())
        s2.wait_stream(torch.cuda.current_stream())
        for _ in range(20):
            if mode in ("h2d", "both"):
                with torch.cuda.stream(s1):
                    d1.copy_(hi, non_blocking=True)
            if mode in ("d2h", "both"):
                with torch.cuda.stream(s2):
                    ho.copy_(d2, non_blocking=True)
        torch.cuda.current_stream().wait_stream(s1)
        torch.cuda.current_stream().wait_stream(s2)
        e1.record()
        torch.cuda.synchronize()
        res[mode] = e0.elapsed_time(e1) / 20
out = [None] * world
if world > 1:
    dist.all_gather_object(out, res)
else:
    out = [res]
if rank == 0:
    for r, x in enumerate(out):
        print(r, {k: f"{v:.3f} ms ({mb * 2**20 / (v * 1e-3) / 1e9:.1f} GB/s)" for k, v in x.items()})
if world > 1:
    dist.destroy_process_group()
