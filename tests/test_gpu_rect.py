"""Rectangular grids (nx != nz), partial tiles in both directions, sources and
receivers next to tile borders: both engines and every history store against
the float64 oracle, with and without density.  The BASELINE configs and the
reference's own cases are all square, so an x/z mix-up in tile indexing, tensor
map strides or the ring-strip layout would otherwise go unseen."""

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


def _rect_case(nx, nz, pml, rho, nt=260, seed=7):
    dx, dt, f_c = 1e-4, 2e-8, 1.5e6
    rng = np.random.default_rng(seed)
    grid = pk.Grid2D(nx, nz, dx, dt, nt)
    damp = pk.build_pml(grid, pml)
    # a linear array along z on the first undamped row + 1, every 3rd column; 3 transmits
    cols = np.arange(pml + 2, nz - pml - 2, 3)
    nodes = np.stack([np.full(cols.shape, pml + 1), cols], axis=1)
    tx = np.array([0, len(cols) // 2, len(cols) - 1])
    rx = np.broadcast_to(np.arange(len(cols)), (3, len(cols))).copy()
    geom = pk.AcquisitionGeometry(grid, nodes, rx, 0.0, tx_elements=tx)
    t = np.arange(nt) * dt
    t0 = 2.0 / f_c
    pulse = pk.SourcePulse(np.sin(2 * np.pi * f_c * (t - t0)) * np.exp(-((t - t0) * f_c) ** 2),
                           dt, f_c)
    c = np.full((nx, nz), 1540.0)
    xx, zz = np.meshgrid(np.arange(nx), np.arange(nz), indexing="ij")
    for _ in range(3):  # inclusions, one of them straddling a tile border (x = 32 / z = 64)
        cx, cz = rng.integers(pml + 8, nx - pml - 8), rng.integers(pml + 8, nz - pml - 8)
        c[(xx - cx) ** 2 + (zz - cz) ** 2 <= rng.integers(3, 7) ** 2] += rng.uniform(-40, 40)
    c[28:37, 60:69] += 25.0
    r = None
    if rho:
        r = np.full((nx, nz), 1000.0)
        r[(xx - nx // 2) ** 2 + (zz - nz // 2) ** 2 <= 64] = 1080.0
        r[28:37, 60:69] = 960.0
    return grid, geom, pulse, damp, c, r


@pytest.mark.parametrize("shape", [(72, 104), (104, 72), (40, 200)])
@pytest.mark.parametrize("rho", [False, True])
def test_rectangular_grid_vs_oracle(gpu, shape, rho):
    nx, nz = shape
    grid, geom, pulse, damp, c_true, r = _rect_case(nx, nz, 6, rho)
    tx, rx = geom.tx_nodes(), geom.rx_nodes()
    obs, _ = oracle.forward_sweep(c_true, damp.values, grid.dx, grid.dt, pulse.samples, tx, rx, rho=r)
    c0 = np.full(grid.shape, 1520.0)
    m_ref, g_ref, tr_ref = oracle.misfit_gradient(c0, damp.values, grid.dx, grid.dt, pulse.samples,
                                                  tx, rx, obs, geom.element_nodes, rho=r)
    engines = ("stepwise",) if rho else ("stepwise", "cluster")
    for engine in engines:
        eng = fwd.get_engine(grid, tx, rx, geom.element_nodes, pulse.samples, damp,
                             has_rho=rho, engine=engine)
        if engine == "stepwise":
            assert eng.info()["stepwise_kernels"] == "tile"
        eng.set_model(c_true[None], None if r is None else r[None])
        assert rel_l2(eng.forward().cpu().numpy(), obs) <= TOL, engine
        eng.set_model(c0[None], None if r is None else r[None])
        stores = ("strips", "full", "checkpoint") if engine == "stepwise" else ("strips", "full", "lap")
        for store in stores:
            mis, g, tr = eng.misfit_and_gradient(torch.as_tensor(obs).to(gpu), store=store,
                                                 return_traces=True)
            assert eng.last_engine == engine
            assert rel_l2(tr.cpu().numpy(), tr_ref) <= TOL, (engine, store)
            assert rel_l2(g[0].cpu().numpy(), g_ref) <= TOL, (engine, store)
            assert abs(float(mis[0]) - m_ref) <= TOL * m_ref, (engine, store)


def test_rectangular_grid_poisoned_workspace(gpu):
    """No kernel may read workspace memory it did not write: with the allocator's
    recycled blocks NaN-filled before the engine takes them (field buffers,
    strips, receiver samples, accumulators all come from there), the stepwise
    tile kernels and the cluster engine still match the oracle."""
    grid, geom, pulse, damp, c_true, r = _rect_case(72, 104, 6, True)
    tx, rx = geom.tx_nodes(), geom.rx_nodes()
    obs, _ = oracle.forward_sweep(c_true, damp.values, grid.dx, grid.dt, pulse.samples, tx, rx, rho=r)
    c0 = np.full(grid.shape, 1520.0)
    m_ref, g_ref, _ = oracle.misfit_gradient(c0, damp.values, grid.dx, grid.dt, pulse.samples, tx, rx,
                                             obs, geom.element_nodes, rho=r)
    for store in ("strips", "full", "checkpoint"):
        fwd._ENGINE_CACHE.clear()
        torch.cuda.synchronize()
        torch.cuda.empty_cache()
        junk = torch.full((1 << 27,), float("nan"), device=gpu)  # 512 MiB of NaN
        del junk
        eng = fwd.get_engine(grid, tx, rx, geom.element_nodes, pulse.samples, damp, has_rho=True,
                             engine="stepwise")
        eng.set_model(c0[None], r[None])
        mis, g = eng.misfit_and_gradient(torch.as_tensor(obs).to(gpu), store=store)
        assert torch.isfinite(g).all(), store
        assert rel_l2(g[0].cpu().numpy(), g_ref) <= TOL, store
        assert abs(float(mis[0]) - m_ref) <= TOL * m_ref, store
