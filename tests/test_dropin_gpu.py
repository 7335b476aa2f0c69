"""The drop-in inside the UNMODIFIED reference: its own AggregationRegion and
task::Scheduler drive make_stage_kernel_gpu (include/tmgpu_taskmesh.hpp);
outputs equal make_stage_kernel bitwise for max_slices 1/3/8/40 and a
non-finite slice fails all four promises of its fused batch."""
import os
import subprocess

import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu


def test_dropin_inside_reference_aggregation_region():
    exe = os.path.join(O.REF_DIR, "dropin_test")
    if not os.path.exists(exe):
        pytest.skip("oracle/_ref/dropin_test not built (needs /root/reference at build time)")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "DROPIN_OK" in r.stdout
    lines = [l for l in r.stdout.splitlines() if "error batch" in l]
    assert len(lines) == 2 and all("4/4 promises failed: non-finite state" in l for l in lines)
    assert lines[0].split("failed:")[1] == lines[1].split("failed:")[1]  # same SolverError text
