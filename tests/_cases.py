"""Shared builders for the parity tests (inputs only; the oracle is imported by tests)."""

from __future__ import annotations

import numpy as np

from paper_2603_04070_b200 import configs
import paper_2603_04070_b200 as pk

from .conftest import GOLDEN


def rel_l2(a, b) -> float:
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def ring48():
    z = np.load(GOLDEN / "ring48.npz")
    grid = pk.Grid2D(48, 48, float(z["dx"]), float(z["dt"]), z["pulse"].shape[0])
    geom = pk.AcquisitionGeometry(grid, z["nodes"], z["rx_pattern"], 0.028)
    pulse = pk.SourcePulse(z["pulse"], grid.dt, 2e5)
    damp = pk.build_pml(grid, 8)
    return z, grid, geom, pulse, damp


def gradcheck16():
    z = np.load(GOLDEN / "gradcheck16.npz")
    grid = pk.Grid2D(16, 16, float(z["dx"]), float(z["dt"]), z["pulse"].shape[0])
    geom = pk.AcquisitionGeometry(grid, z["nodes"], z["rx_pattern"], 0.010)
    pulse = pk.SourcePulse(z["pulse"], grid.dt, 3e5)
    return z, grid, geom, pulse


def config_setup(cfg: int, seed: int = 0, n_phantoms=None):
    """(workload, grid, geometry, pulse, damping) for a BASELINE config."""
    wl = configs.make_workload(cfg, seed=seed, n_phantoms=n_phantoms)
    s = wl.spec
    grid = pk.Grid2D(s.n, s.n, s.dx, s.dt, s.nt)
    geom = pk.AcquisitionGeometry(grid, wl.nodes, wl.rx, 0.0, tx_elements=wl.tx)
    pulse = pk.SourcePulse(wl.pulse, s.dt, s.f_c)
    damp = pk.build_pml(grid, s.pml)
    return wl, grid, geom, pulse, damp


def small_linear(n=40, pml=6, nt=260, n_el=12, n_tx=3, seed=3, rho=False, dx=1e-4, dt=2e-8,
                 f_c=1.5e6):
    """Small linear-array case (config-0 conventions) the oracle finishes in seconds."""
    spec = configs.WorkloadSpec("small", n, pml, dx, dt, nt, f_c, n_el, n_tx, None, n_el, 1, 0,
                                (2, 2), "ellipse", (3.0, 6.0), 40.0, rho, 0.0)
    wl = configs.make_workload(spec, seed=seed)
    N = spec.n
    grid = pk.Grid2D(N, N, dx, dt, nt)
    geom = pk.AcquisitionGeometry(grid, wl.nodes, wl.rx, 0.0, tx_elements=wl.tx)
    pulse = pk.SourcePulse(wl.pulse, dt, f_c)
    damp = pk.build_pml(grid, pml)
    return wl, grid, geom, pulse, damp
