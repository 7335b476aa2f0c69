"""Kernel-level FMM gravity timing (uniform level D) for ncu runs."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2412_15518_b200.gravity import GravitySolver
D = int(sys.argv[1]) if len(sys.argv) > 1 else 7
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
G = GravitySolver(D)
n3 = (1 << D) ** 3
m = torch.rand(n3, dtype=torch.float64, device="cuda") / n3
for _ in range(2):
    G.solve(m)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    G.solve(m)
e1.record()
torch.cuda.synchronize()
print("D", D, "ms/solve", e0.elapsed_time(e1) / reps)
