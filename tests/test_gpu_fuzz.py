"""Seeded random small cases against the float64 oracle: grid shapes from a few
cells to several tiles (any nz % 4, incl. nz % 4 != 0 which leaves the tile
kernels), PML thickness 0..10 (0: no damping, the strip ring lies outside the
grid), random transmit / receive nodes anywhere in the undamped region (tile
corners, duplicates across shots), density on/off, both engines, every store."""

from __future__ import annotations

import numpy as np
import pytest
import torch

import oracle
import paper_2603_04070_b200 as pk
from paper_2603_04070_b200 import forward as fwd

from ._cases import rel_l2

pytestmark = pytest.mark.gpu

TOL = 1e-4


def _case(seed):
    rng = np.random.default_rng(1000 + seed)
    nx = int(rng.choice([20, 33, 48, 70, 97]))
    nz = int(rng.choice([24, 36, 64, 68, 130, 41]))
    pml = int(rng.choice([0, 4, 7, 10]))
    if 2 * pml + 8 > min(nx, nz):
        pml = 0
    nt = int(rng.integers(120, 220))
    rho = bool(rng.integers(0, 2))
    dx, dt, f_c = 1e-4, 2e-8, 1.5e6
    grid = pk.Grid2D(nx, nz, dx, dt, nt)
    damp = pk.build_pml(grid, pml)
    lo, hx, hz = pml + 1, nx - pml - 2, nz - pml - 2
    n_el = int(rng.integers(4, 10))
    nodes = np.unique(np.stack([rng.integers(lo, hx + 1, n_el), rng.integers(lo, hz + 1, n_el)], 1),
                      axis=0)
    n_el = len(nodes)
    S = int(rng.integers(1, min(4, n_el) + 1))
    tx = rng.choice(n_el, S, replace=False)
    R = int(rng.integers(1, n_el + 1))
    rx = np.stack([rng.choice(n_el, R, replace=False) for _ in range(S)])
    geom = pk.AcquisitionGeometry(grid, nodes, rx, 0.0, tx_elements=tx)
    t = np.arange(nt) * dt
    t0 = 2.0 / f_c
    pulse = pk.SourcePulse(np.sin(2 * np.pi * f_c * (t - t0)) * np.exp(-((t - t0) * f_c) ** 2), dt, f_c)
    xx, zz = np.meshgrid(np.arange(nx), np.arange(nz), indexing="ij")
    c = np.full((nx, nz), 1540.0)
    for _ in range(3):
        cx, cz = rng.integers(0, nx), rng.integers(0, nz)
        c[(xx - cx) ** 2 + (zz - cz) ** 2 <= rng.integers(2, 8) ** 2] += rng.uniform(-50, 50)
    r = None
    if rho:
        r = np.full((nx, nz), 1000.0)
        r[(xx - nx // 2) ** 2 + (zz - nz // 3) ** 2 <= 30] = rng.uniform(950, 1100)
        r[:3, :] = 1050.0  # density contrast on the grid edge: the outer faces
        r[:, -2:] = 970.0
    return grid, geom, pulse, damp, c, r


@pytest.mark.parametrize("seed", range(24))
def test_random_case_vs_oracle(gpu, seed):
    grid, geom, pulse, damp, c_true, r = _case(seed)
    tx, rx = geom.tx_nodes(), geom.rx_nodes()
    obs, _ = oracle.forward_sweep(c_true, damp.values, grid.dx, grid.dt, pulse.samples, tx, rx, rho=r)
    c0 = np.full(grid.shape, 1515.0)
    m_ref, g_ref, tr_ref = oracle.misfit_gradient(c0, damp.values, grid.dx, grid.dt, pulse.samples,
                                                  tx, rx, obs, geom.element_nodes, rho=r)
    rr = None if r is None else r[None]
    for engine in ("stepwise", "auto"):
        eng = fwd.get_engine(grid, tx, rx, geom.element_nodes, pulse.samples, damp,
                             has_rho=r is not None, engine=engine)
        if engine == "stepwise":
            assert eng.info()["stepwise_kernels"] == ("tile" if grid.nz % 4 == 0 else "stream")
        eng.set_model(c_true[None], rr)
        assert rel_l2(eng.forward().cpu().numpy(), obs) <= TOL, (seed, engine)
        eng.set_model(c0[None], rr)
        for store in ("auto", "strips", "full", "checkpoint"):
            if store == "checkpoint" and engine != "stepwise":
                continue
            mis, g, tr = eng.misfit_and_gradient(torch.as_tensor(obs).to(gpu), store=store,
                                                 return_traces=True)
            assert rel_l2(tr.cpu().numpy(), tr_ref) <= TOL, (seed, engine, store)
            assert rel_l2(g[0].cpu().numpy(), g_ref) <= TOL, (seed, engine, store, eng.last_engine)
            assert abs(float(mis[0]) - m_ref) <= TOL * max(m_ref, 1e-30), (seed, engine, store)
