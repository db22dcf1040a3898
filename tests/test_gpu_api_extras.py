"""The rest of the reference's public forward/gradient API surface on the device:
laplacian (forward.py:211-223), step_wavefield (forward.py:237-253),
fd_gradient_oracle (adjoint.py:154-186), and the failure semantics of the
unfolded inference (per-stage CFL check, adjoint.py:105 -> forward.py:259-263)
and of the batched/engine entry points (shape checks)."""

from __future__ import annotations

import numpy as np
import pytest
import torch

import oracle
import paper_2603_04070_b200 as pk
from paper_2603_04070_b200 import forward as fwd
from paper_2603_04070_b200.network import make_update_nets

from ._cases import gradcheck16, rel_l2, ring48

pytestmark = pytest.mark.gpu


def test_laplacian_bit_identical_to_reference_order(gpu):
    rng = np.random.default_rng(0)
    u = rng.standard_normal((3, 37, 41))
    got = pk.laplacian(u, 1e-4)
    assert got.dtype == np.float64 and got.shape == u.shape
    assert np.array_equal(got, oracle.lap5(u, 1e-4))  # oracle.lap5 == forward.laplacian bits
    assert np.array_equal(pk.laplacian(u[0], 2.5e-3), oracle.lap5(u[0], 2.5e-3))


def test_step_wavefield_bit_identical_and_checks(gpu):
    z, grid, geom, pulse, damp = ring48()
    rng = np.random.default_rng(1)
    u1 = rng.standard_normal(grid.shape)
    u2 = rng.standard_normal(grid.shape)
    s = np.zeros(grid.shape)
    s[10, 12] = 0.7
    sos = pk.SosMap(grid, z["c_true"])
    got = pk.step_wavefield(u1, u2, sos, damp, s, grid.dt)
    a, b, e = oracle.step_coeffs(sos.values, damp.values, grid.dt)
    want = a * u1 + b * u2 + e * oracle.lap5(u1, grid.dx) + s  # forward.py:253
    assert np.array_equal(got, want)
    with pytest.raises(ValueError, match="shape"):
        pk.step_wavefield(u1[:-1], u2, sos, damp, s, grid.dt)
    bad = u2.copy()
    bad[3, 3] = np.nan
    with pytest.raises(pk.NumericError, match="u_prev2"):
        pk.step_wavefield(u1, bad, sos, damp, s, grid.dt)


def test_fd_gradient_oracle_vs_reference_gradient(gpu):
    """Central differences on the device against the reference's adjoint gradient
    (gradcheck16 = cli.py:212-240).  f32 receiver samples set a noise floor on
    the misfit, so eps = 1 m/s here (truncation error ~(eps/c)^2 ~ 4e-7)."""
    z, grid, geom, pulse = gradcheck16()
    obs = pk.ChannelData(z["obs"], geom, grid.dt)
    c0 = pk.SosMap(grid, z["c0"])
    cells = [tuple(c) for c in z["cells"]]
    fd = pk.fd_gradient_oracle(c0, obs, pulse, cells, eps=1.0)
    g_ref = z["grad"][z["cells"][:, 0], z["cells"][:, 1]]
    rel = np.abs(fd - g_ref) / np.abs(g_ref)
    assert rel.max() <= 2e-3, rel
    with pytest.raises(ValueError):
        pk.fd_gradient_oracle(c0, obs, pulse, cells, eps=0.0)


def test_unfold_infer_raises_cfl_per_stage(gpu):
    """With clamp bounds above the CFL limit, the stage whose input map violates
    it raises the reference's ValueError (no unstable sweep result returned)."""
    z, grid, geom, pulse, damp = ring48()
    obs = pk.ChannelData(z["obs"], geom, grid.dt)
    limit = grid.dx / (grid.dt * np.sqrt(2.0))
    nets = make_update_nets(2, seed=1, device=gpu)
    for n in nets:  # the first stage's update pushes every cell far above the limit
        with torch.no_grad():
            last = n.body[-1]
            last.weight.zero_()
            last.bias.fill_(10.0)
    setup = pk.InversionSetup(pulse, damp, (1300.0, 2.0 * limit))
    with pytest.raises(ValueError, match="CFL violated"):
        pk.unfold_infer(obs, pk.homogeneous_map(grid, 1500.0), nets, setup)
    # within the limit the same call runs
    ok = pk.InversionSetup(pulse, damp, (1300.0, 0.999 * limit))
    out = pk.unfold_infer(obs, pk.homogeneous_map(grid, 1500.0), nets, ok)
    assert len(out) == 2


def test_shape_checks_of_engine_and_batch(gpu):
    z, grid, geom, pulse, damp = ring48()
    eng = fwd.get_engine(grid, geom.tx_nodes(), geom.rx_nodes(), geom.element_nodes,
                         pulse.samples, damp)
    eng.set_model(z["c0"][None])
    obs = torch.as_tensor(z["obs"]).to(gpu)
    with pytest.raises(ValueError, match="observed data shape"):
        eng.misfit_and_gradient(obs[:-1])
    with pytest.raises(ValueError, match="observed data shape"):
        eng.misfit_and_gradient(obs[:, :, :-1])
    c = pk.SosMap(grid, z["c0"])
    o = pk.ChannelData(z["obs"], geom, grid.dt)
    with pytest.raises(ValueError):
        pk.misfit_and_gradient_batch([c, c], [o], pulse, damp)
    other = pk.AcquisitionGeometry(grid, geom.element_nodes, geom.rx_pattern[:, ::-1].copy(),
                                   geom.diameter)
    o2 = pk.ChannelData(z["obs"], other, grid.dt)
    with pytest.raises(ValueError, match="geometry"):
        pk.misfit_and_gradient_batch([c, c], [o, o2], pulse, damp)
    mis, gs = pk.misfit_and_gradient_batch([c, c], [o, o], pulse, damp)
    m1, g1 = pk.misfit_and_gradient(c, o, pulse, damp)
    assert mis[0] == m1 and np.array_equal(gs[1].values, g1.values)


def test_public_api_arith_keyword(gpu):
    """simulate_all / misfit_and_gradient take arith="f64": the float64 sweep sits an
    order of magnitude closer to the reference than the default f32 one, both inside
    the parity bars; an unknown value raises."""
    z, grid, geom, pulse, damp = ring48()
    c_true, c0 = pk.SosMap(grid, z["c_true"]), pk.SosMap(grid, z["c0"])
    obs = pk.ChannelData(z["obs"], geom, grid.dt)
    e32 = rel_l2(pk.simulate_all(c_true, geom, pulse, damp).traces, z["obs"])
    e64 = rel_l2(pk.simulate_all(c_true, geom, pulse, damp, arith="f64").traces, z["obs"])
    assert e64 < 1e-7 < e32 <= 1e-4
    for arith in ("f32", "f64"):
        m, g = pk.misfit_and_gradient(c0, obs, pulse, damp, arith=arith)
        assert rel_l2(g.values, z["grad"]) <= 1e-4
        assert abs(m - float(z["misfit"])) <= 1e-4 * float(z["misfit"])
    with pytest.raises(ValueError, match="arith"):
        pk.compute_gradient(c0, obs, pulse, damp, arith="bf16")
