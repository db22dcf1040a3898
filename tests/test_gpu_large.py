"""Parity at BASELINE.json's larger configs (stepwise engine, boundary strips).

Sizes the float64 oracle can finish on the host are checked directly (config 2
with variable density at full nt on 2 shots; config 3's grid on 1 shot with a
shortened time axis); at config 4's full size (1088^2, nt 6000) the checks are
size-independent properties: zero residual -> zero gradient, linearity in the
residual, and strip reconstruction vs full-history storage."""

from __future__ import annotations

import dataclasses

import numpy as np
import pytest
import torch

import oracle
import paper_2603_04070_b200 as pk
from paper_2603_04070_b200 import configs
from paper_2603_04070_b200 import forward as fwd

from ._cases import rel_l2

pytestmark = pytest.mark.gpu


def _setup(cfg, n_shots, nt=None, seed=0):
    spec = configs.get_config(cfg)
    if nt:
        spec = dataclasses.replace(spec, nt=nt)
    wl = configs.make_workload(spec, seed=seed, n_phantoms=1)
    sel = np.linspace(0, len(wl.tx) - 1, n_shots).round().astype(int)
    tx, rxp = wl.tx[sel], wl.rx[sel]
    grid = pk.Grid2D(spec.n, spec.n, spec.dx, spec.dt, spec.nt)
    geom = pk.AcquisitionGeometry(grid, wl.nodes, rxp, 0.0, tx_elements=tx)
    damp = pk.build_pml(grid, spec.pml)
    return wl, grid, geom, damp


def _eng(grid, geom, wl, damp, engine="stepwise"):
    return fwd.get_engine(grid, geom.tx_nodes(), geom.rx_nodes(), geom.element_nodes, wl.pulse,
                          damp, has_rho=wl.rho is not None, engine=engine)


def test_config2_density_full_nt_vs_oracle(gpu):
    wl, grid, geom, damp = _setup(2, 2)
    rho = wl.rho[0]
    tx, rx = geom.tx_nodes(), geom.rx_nodes()
    obs, _ = oracle.forward_sweep(wl.c_true[0], damp.values, grid.dx, grid.dt, wl.pulse, tx, rx, rho=rho)
    c0 = np.full(grid.shape, 1540.0)
    m_ref, g_ref, tr_ref = oracle.misfit_gradient(c0, damp.values, grid.dx, grid.dt, wl.pulse, tx, rx,
                                                  obs, geom.element_nodes, rho=rho)
    eng = _eng(grid, geom, wl, damp)
    eng.set_model(wl.c_true, wl.rho)
    assert rel_l2(eng.forward().cpu().numpy(), obs) <= 1e-4
    eng.set_model(c0[None], wl.rho)
    mis, g = eng.misfit_and_gradient(torch.as_tensor(obs).to(gpu))
    assert eng.last_engine == "stepwise"
    assert rel_l2(g[0].cpu().numpy(), g_ref) <= 1e-4
    assert abs(float(mis[0]) - m_ref) <= 1e-4 * m_ref


def test_config3_grid_one_shot_vs_oracle(gpu):
    wl, grid, geom, damp = _setup(3, 1, nt=700)
    tx, rx = geom.tx_nodes(), geom.rx_nodes()
    rho = wl.rho[0]
    obs, _ = oracle.forward_sweep(wl.c_true[0], damp.values, grid.dx, grid.dt, wl.pulse, tx, rx, rho=rho)
    c0 = np.full(grid.shape, 1540.0)
    m_ref, g_ref, _ = oracle.misfit_gradient(c0, damp.values, grid.dx, grid.dt, wl.pulse, tx, rx, obs,
                                             geom.element_nodes, rho=rho)
    eng = _eng(grid, geom, wl, damp)
    eng.set_model(c0[None], wl.rho)
    for store in ("strips", "full"):
        mis, g = eng.misfit_and_gradient(torch.as_tensor(obs).to(gpu), store=store)
        assert rel_l2(g[0].cpu().numpy(), g_ref) <= 1e-4, store


def test_config4_full_size_properties(gpu):
    wl, grid, geom, damp = _setup(4, 2)
    assert grid.nx == 1088 and grid.nt == 6000
    eng = _eng(grid, geom, wl, damp)
    eng.set_model(wl.c_true, wl.rho)
    tr = eng.forward().double()
    assert torch.isfinite(tr).all() and float(tr.abs().max()) > 0
    c0 = np.full((1,) + grid.shape, 1540.0)
    eng.set_model(c0, wl.rho)
    # zero residual -> zero gradient
    own = eng.forward().double()
    mis0, g0 = eng.misfit_and_gradient(own)
    assert float(mis0[0]) == 0.0 and float(g0.abs().max()) == 0.0
    # linearity in the residual (the adjoint is linear; f32 state only rounds)
    r = tr - own
    _, g1 = eng.misfit_and_gradient(own - r)
    _, g2 = eng.misfit_and_gradient(own - 2 * r)
    assert rel_l2(g2.cpu().numpy(), 2 * g1.cpu().numpy()) <= 1e-5


def test_config4_grid_strips_vs_full_history(gpu):
    wl, grid, geom, damp = _setup(4, 1, nt=1500)
    eng = _eng(grid, geom, wl, damp)
    eng.set_model(wl.c_true, wl.rho)
    obs = eng.forward().double()
    eng.set_model(np.full((1,) + grid.shape, 1540.0), wl.rho)
    _, gs = eng.misfit_and_gradient(obs, store="strips")
    _, gf = eng.misfit_and_gradient(obs, store="full")
    assert rel_l2(gs.cpu().numpy(), gf.cpu().numpy()) <= 1e-5
