"""The aggregation executor of this repo (csrc/aggregator.cpp: tmgpu_region_*,
the CUDA-stream AggregationRegion mirror) on the same workload as
oracle/dropin/dropin_bench.cpp: `count` Euler slices (the C3 leaf count)
submitted from the host, one aggregated launch per batch; cell-stage/s per
max_slices. Prints JSON lines."""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2412_15518_b200 import aggregator as A  # noqa: E402
from paper_2412_15518_b200 import hydro as H  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 5888
g = H.StageGeom(vars=5)
rng = np.random.default_rng(2412518)
S = 12 ** 3
slices = np.zeros((n, g.in_slice()))
for s in range(n):
    dx = (1.0 / 256) * (1 + s % 2)
    H.encode_header(H.StageParams(H.Mode.euler, dx, 0.2 * dx), slices[s])
    rho, p = rng.uniform(0.2, 2.0, S), rng.uniform(0.2, 2.0, S)
    u, v, w = (rng.uniform(-0.5, 0.5, S) for _ in range(3))
    slices[s, 8:] = np.concatenate([rho, rho * u, rho * v, rho * w, p / 0.4 + 0.5 * rho * (u * u + v * v + w * w)])
for ms in (8, 64, 512, n):
    best = 1e30
    for _ in range(3):
        execs = A.ExecutorPool(4)
        cnt = A.AggCounters()
        t0 = time.perf_counter()
        region = A.AggregationRegion(execs, g, ms, n, cnt)
        futs = [region.submit_slice(slices[s]) for s in range(n)]
        region.flush()
        A.when_all(futs)
        best = min(best, time.perf_counter() - t0)
        region.close()
    print(json.dumps({"path": "gpu", "api": "paper_2412_15518_b200.aggregator.AggregationRegion(StageGeom)",
                      "max_slices": ms, "slices": n, "launches": cnt.launches, "seconds": best,
                      "cell_stage_per_s": n * 512 / best,
                      "slice_GBps": n * (g.in_slice() + g.out_slice()) * 8 / best / 1e9}), flush=True)
