"""SPEC properties of the scheme (the usable known-answer tests of
SURVEY §8(c)) on the CUDA path, both engines: zero-field fixed point, source
linearity, shot additivity of misfit and gradient, point-to-point reciprocity,
linearity of the gradient in the residual.  The float64 oracle has the same
tests in tests/test_oracle_properties.py; here the bounds are those of f32
storage."""

from __future__ import annotations

import numpy as np
import pytest
import torch

import paper_2603_04070_b200 as pk
from paper_2603_04070_b200 import forward as fwd

from ._cases import rel_l2, small_linear

pytestmark = pytest.mark.gpu

ENGINES = ("cluster", "stepwise")


def _engine(grid, geom, pulse, damp, engine):
    return fwd.get_engine(grid, geom.tx_nodes(), geom.rx_nodes(), geom.element_nodes,
                          pulse.samples, damp, engine=engine)


@pytest.mark.parametrize("engine", ENGINES)
def test_zero_source_gives_zero_traces(gpu, engine):
    wl, grid, geom, pulse, damp = small_linear(seed=4)
    eng = _engine(grid, geom, pk.SourcePulse(np.zeros_like(pulse.samples), grid.dt, pulse.f_c),
                  damp, engine)
    eng.set_model(wl.c_true)
    tr = eng.forward()
    assert eng.last_engine == engine
    assert not bool(tr.any())


@pytest.mark.parametrize("engine", ENGINES)
def test_source_linearity(gpu, engine):
    """Traces scale with the pulse: exactly for a power of two (every operation of
    the sweep is linear and the scaling commutes with rounding), to f32 rounding
    otherwise."""
    wl, grid, geom, pulse, damp = small_linear(seed=5)
    out = {}
    for k in (1.0, 2.0, 2.5):
        eng = _engine(grid, geom, pk.SourcePulse(k * pulse.samples, grid.dt, pulse.f_c), damp, engine)
        eng.set_model(wl.c_true)
        out[k] = eng.forward().double().cpu().numpy()
    assert np.abs(out[1.0]).max() > 0
    assert np.array_equal(out[2.0], 2.0 * out[1.0])
    assert rel_l2(out[2.5], 2.5 * out[1.0]) <= 2e-6


@pytest.mark.parametrize("engine", ENGINES)
@pytest.mark.parametrize("store", ("full", "strips"))
def test_shot_additivity(gpu, engine, store):
    """Misfit and gradient of all transmits = the sums over single transmits."""
    wl, grid, geom, pulse, damp = small_linear(seed=6)
    eng = _engine(grid, geom, pulse, damp, engine)
    eng.set_model(wl.c_true)
    obs = eng.forward().double() * 1.01
    m_all, g_all = eng.misfit_and_gradient(obs, store=store)
    m_sum = torch.zeros_like(m_all)
    g_sum = torch.zeros_like(g_all)
    for u in range(eng.n_units):
        m, g = eng.misfit_and_gradient(obs, store=store, units=(u, u + 1))
        m_sum += m
        g_sum += g
    assert float(g_all.abs().max()) > 0
    assert rel_l2(g_sum.cpu().numpy(), g_all.cpu().numpy()) <= 1e-6
    assert abs(float(m_sum[0]) - float(m_all[0])) <= 1e-12 * float(m_all[0])


@pytest.mark.parametrize("engine", ENGINES)
def test_reciprocity(gpu, engine):
    """E L is self-adjoint in the 1/E-weighted inner product: a -> b equals b -> a
    when both nodes see the same speed."""
    wl, grid, geom, pulse, damp = small_linear(seed=7)
    el = np.asarray(geom.element_nodes)
    a, b = el[1], el[-2]
    c = np.array(wl.c_true[0])
    c[a[0], a[1]] = c[b[0], b[1]] = 1540.0
    tr = []
    for src, rcv in ((a, b), (b, a)):
        g = pk.AcquisitionGeometry(grid, np.stack([src, rcv]), np.array([[1]]), 0.0,
                                   tx_elements=np.array([0]))
        eng = _engine(grid, g, pulse, damp, engine)
        eng.set_model(c[None])
        tr.append(eng.forward().double().cpu().numpy())
    assert np.abs(tr[0]).max() > 0
    assert rel_l2(tr[1], tr[0]) <= 5e-6


@pytest.mark.parametrize("engine", ENGINES)
def test_gradient_linear_in_residual(gpu, engine):
    wl, grid, geom, pulse, damp = small_linear(seed=8)
    eng = _engine(grid, geom, pulse, damp, engine)
    eng.set_model(wl.c_true)
    tr = eng.forward().double()
    r = torch.as_tensor(np.random.default_rng(2).standard_normal(tuple(tr.shape)) * 1e-3,
                        device=tr.device) * tr.abs().max()
    _, g1 = eng.misfit_and_gradient(tr - r)
    _, g2 = eng.misfit_and_gradient(tr - 2.0 * r)
    assert float(g1.abs().max()) > 0
    assert rel_l2(g2.cpu().numpy(), 2.0 * g1.cpu().numpy()) <= 1e-5


def test_config0_full_size_linearity_and_additivity(gpu):
    """The same properties at BASELINE config 0's stated size (160^2, nt 1000, 8 transmits)."""
    from ._cases import config_setup

    wl, grid, geom, pulse, damp = config_setup(0)
    eng = _engine(grid, geom, pulse, damp, "auto")
    eng.set_model(wl.c_true)
    tr = eng.forward().double()
    eng2 = _engine(grid, geom, pk.SourcePulse(2.0 * pulse.samples, grid.dt, pulse.f_c), damp, "auto")
    eng2.set_model(wl.c_true)
    # not bit for bit here: the leading edge of the wavefront passes through the f32
    # subnormal range (first at t = 22, values ~1e-39), where rounding is absolute; one
    # rounding that differs decorrelates the later ones, so the two runs differ by
    # their rounding noise (measured 1e-7 of the peak, the same on both engines)
    tr2 = eng2.forward().double()
    assert rel_l2(tr2.cpu().numpy(), 2.0 * tr.cpu().numpy()) <= 2e-6
    eng.set_model(np.full((1,) + grid.shape, 1540.0))
    m_all, g_all = eng.misfit_and_gradient(tr)
    g_sum = torch.zeros_like(g_all)
    m_sum = 0.0
    for u in range(eng.n_units):
        m, g = eng.misfit_and_gradient(tr, units=(u, u + 1))
        g_sum += g
        m_sum += float(m[0])
    assert float(g_all.abs().max()) > 0
    assert rel_l2(g_sum.cpu().numpy(), g_all.cpu().numpy()) <= 1e-6
    assert abs(m_sum - float(m_all[0])) <= 1e-12 * float(m_all[0])
