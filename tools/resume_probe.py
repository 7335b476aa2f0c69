"""Probe: how far a run resumed from interior-only state (or the current
arena's ghosted grids) drifts from the uninterrupted run after one step."""
import numpy as np
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2412_15518_b200 import amr  # noqa: E402
from paper_2412_15518_b200.driver import HydroDriver
def mk():
    f = amr.build_scenario(amr.Scenario.rotating_star, 2, 4); f.alloc(); return f
f = mk(); f.set_interior(f.scenario_state(amr.Scenario.rotating_star)); d = HydroDriver(f)
for _ in range(2): d.step()
grids = f.get_grids(); inter = f.get_interior()
for mode in ("interior", "grids", "grids+fill"):
    g = mk()
    if mode == "interior": g.set_interior(inter)
    else: g.set_grids(grids)
    if mode == "grids+fill": g.fill_ghosts()
    HydroDriver(g).step()
    if mode == "interior": d.step(); ref = f.get_interior()
    a = g.get_interior()
    print(mode, float((np.abs(a-ref)/np.abs(ref).max(axis=(0,2),keepdims=True)).max()), float((a==ref).mean()))
