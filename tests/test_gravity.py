"""FMM gravity: our specification (oracle/gravity_oracle.c, parity unpinned —
the reference has no gravity code) checked against direct O(N^2)
summation and conservation laws on CPU; the sm_100a kernels must equal the
specification bitwise."""
import ctypes as C

import numpy as np
import pytest

from oracle import oracle as O

dp = C.POINTER(C.c_double)


def _lib():
    L = O.Oracle().lib
    for f in (L.tmo_grav_solve, L.tmo_grav_direct):
        f.argtypes = [C.c_int, dp, dp, dp]
    return L


def _run(f, D, m):
    n3 = (1 << D) ** 3
    phi, g = np.zeros(n3), np.zeros(3 * n3)
    f(D, m.ctypes.data_as(dp), phi.ctypes.data_as(dp), g.ctypes.data_as(dp))
    return phi, g.reshape(3, -1)


def star_masses(D, R=0.3):
    N = 1 << D
    x = (np.arange(N) + 0.5) / N
    Z, Y, X = np.meshgrid(x, x, x, indexing="ij")
    rho = np.maximum(1 - ((X - .5) ** 2 + (Y - .5) ** 2 + (Z - .5) ** 2) / R ** 2, 0) ** 1.5 + 1e-3
    h = 1.0 / N
    return np.ascontiguousarray((rho * (h * h * h)).ravel()), np.stack([X.ravel(), Y.ravel(), Z.ravel()])


@pytest.mark.parametrize("kind", ["star", "random"])
def test_fmm_vs_direct_summation(kind):
    L = _lib()
    D = 4
    m, pos = star_masses(D)
    if kind == "random":
        m = np.random.default_rng(1).uniform(0, 1, m.size) / m.size
    pf, gf = _run(L.tmo_grav_solve, D, m)
    pd, gd = _run(L.tmo_grav_direct, D, m)
    gm = np.sqrt((gd ** 2).sum(0))
    err = np.sqrt(((gf - gd) ** 2).sum(0))
    assert np.max(np.abs(pf - pd) / np.abs(pd)) < 2e-2
    assert np.sqrt(np.mean(err ** 2)) / np.sqrt(np.mean(gm ** 2)) < 4e-2
    F = gf * m  # linear momentum: mutual M2L/P2P forces cancel to round-off
    assert np.abs(F.sum(1)).max() <= 1e-13 * np.abs(F).sum(1).max()


def test_uniform_density_field_points_inward():
    L = _lib()
    D = 3
    N = 8
    m = np.full(N ** 3, 1.0 / N ** 3)
    _, g = _run(L.tmo_grav_solve, D, m)
    x = (np.arange(N) + 0.5) / N - 0.5
    Z, Y, X = np.meshgrid(x, x, x, indexing="ij")
    r = np.stack([X.ravel(), Y.ravel(), Z.ravel()])
    assert ((g * r).sum(0) < 0).all()  # attraction toward the centre


@pytest.mark.gpu
@pytest.mark.parametrize("D", [3, 4, 6])
def test_gpu_fmm_bitwise_equals_specification(D):
    from paper_2412_15518_b200.gravity import GravitySolver

    L = _lib()
    m, _ = star_masses(D)
    m = m * (1 + 1e-3 * np.random.default_rng(D).uniform(-1, 1, m.size))
    pf, gf = _run(L.tmo_grav_solve, D, m)
    phi, g = GravitySolver(D).solve(m)
    assert phi.tobytes() == pf.tobytes()
    assert g.tobytes() == gf.tobytes()


@pytest.mark.gpu
def test_gpu_fmm_from_forest_arena():
    """configs[1]-style: uniform level-4 forest (4,096 leaves, 128^3 cells),
    masses gathered from the device arena."""
    import torch

    from paper_2412_15518_b200 import amr
    from paper_2412_15518_b200.gravity import GravitySolver

    f = amr.build_scenario(amr.Scenario.rotating_star, 4, 4)
    st = f.scenario_state(amr.Scenario.rotating_star)
    f.alloc()
    f.set_interior(st)
    G = GravitySolver(7)
    phi = torch.empty(128 ** 3, dtype=torch.float64, device="cuda")
    g = torch.empty(3 * 128 ** 3, dtype=torch.float64, device="cuda")
    G.solve_forest(f, phi, g)
    # the same masses on the host, placed by leaf coordinates
    h = 1.0 / 128
    m = np.zeros((128, 128, 128))
    for s, p in enumerate(f.local_leaves()):
        _, ci, cj, ck = amr.unpack(int(p))
        m[8 * ck:8 * ck + 8, 8 * cj:8 * cj + 8, 8 * ci:8 * ci + 8] = st[s, 0].reshape(8, 8, 8) * (h * h * h)
    phi2, g2 = GravitySolver(7).solve(np.ascontiguousarray(m.ravel()))
    assert phi.cpu().numpy().tobytes() == phi2.tobytes()
    assert g.cpu().numpy().reshape(3, -1).tobytes() == g2.tobytes()
    F = g2 * m.ravel()
    assert np.abs(F.sum(1)).max() <= 1e-12 * np.abs(F).sum(1).max()
