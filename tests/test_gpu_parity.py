"""GPU parity tests: the sm_100a path (through the C ABI) vs the reference's
golden fixtures and the float64 oracle.  Tolerances from BASELINE.json's
north star: relative L2 <= 1e-4 on fp32 traces and per-iteration gradients,
<= 1e-3 on the final SoS map."""

from __future__ import annotations

import numpy as np
import pytest
import torch

import oracle
import paper_2603_04070_b200 as pk
from paper_2603_04070_b200 import forward as fwd

from ._cases import config_setup, gradcheck16, rel_l2, ring48, small_linear

pytestmark = pytest.mark.gpu

TRACE_TOL = 1e-4
GRAD_TOL = 1e-4
MAP_TOL = 1e-3
ENGINES = ("cluster", "stepwise")
STORES = ("full", "strips")


def _engine(grid, geom, pulse, damp, engine, n_phantoms=1, has_rho=False):
    return fwd.get_engine(grid, geom.tx_nodes(), geom.rx_nodes(), geom.element_nodes,
                          pulse.samples, damp, n_phantoms=n_phantoms, has_rho=has_rho,
                          engine=engine)


@pytest.mark.parametrize("engine", ENGINES)
@pytest.mark.parametrize("store", STORES)
def test_ring48_matches_reference_golden(gpu, engine, store):
    z, grid, geom, pulse, damp = ring48()
    assert np.array_equal(damp.values, z["damping"])
    eng = _engine(grid, geom, pulse, damp, engine)
    eng.set_model(z["c_true"][None])
    tr = eng.forward().cpu().numpy()
    assert rel_l2(tr, z["obs"]) <= TRACE_TOL
    eng.set_model(z["c0"][None])
    mis, g = eng.misfit_and_gradient(torch.as_tensor(z["obs"]).to(gpu), store=store)
    assert eng.last_engine == engine
    assert rel_l2(g[0].cpu().numpy(), z["grad"]) <= GRAD_TOL
    assert abs(float(mis[0]) - float(z["misfit"])) <= 1e-4 * float(z["misfit"])


def test_gradcheck16_no_pml_matches_reference_and_fd(gpu):
    z, grid, geom, pulse = gradcheck16()
    for engine in ENGINES:
        eng = _engine(grid, geom, pulse, pk.zero_damping(grid), engine)
        eng.set_model(z["c0"][None])
        mis, g = eng.misfit_and_gradient(torch.as_tensor(z["obs"]).to(gpu))
        g = g[0].cpu().numpy()
        assert rel_l2(g, z["grad"]) <= GRAD_TOL
        cells = z["cells"]
        fd = z["fd"]
        # the reference's own CLI check (cli.py:212-240) at its tolerance 1e-4
        rel = np.abs(g[cells[:, 0], cells[:, 1]] - fd) / np.abs(fd)
        assert rel.max() < 1e-3


@pytest.mark.parametrize("engine", ENGINES)
@pytest.mark.parametrize("store", STORES)
def test_gradcheck16_poisoned_workspace(gpu, engine, store):
    """No PML puts the strip ring outside the grid; no kernel may read the
    (never written) ring slots — NaN-filled recycled memory must not leak in."""
    z, grid, geom, pulse = gradcheck16()
    fwd._ENGINE_CACHE.clear()
    torch.cuda.synchronize()
    junk = torch.full((1 << 26,), float("nan"), device=gpu)
    del junk
    eng = _engine(grid, geom, pulse, pk.zero_damping(grid), engine)
    eng.set_model(z["c0"][None])
    _, g = eng.misfit_and_gradient(torch.as_tensor(z["obs"]).to(gpu), store=store)
    assert rel_l2(g[0].cpu().numpy(), z["grad"]) <= GRAD_TOL


def test_public_api_ring48(gpu):
    z, grid, geom, pulse, damp = ring48()
    obs = pk.simulate_all(pk.SosMap(grid, z["c_true"]), geom, pulse, damp)
    assert rel_l2(obs.traces, z["obs"]) <= TRACE_TOL
    one = pk.simulate_transmission(pk.SosMap(grid, z["c_true"]), geom, pulse, 3, damp)
    assert one.shape == (grid.nt, geom.n_r)
    assert rel_l2(one, z["obs"][3].T) <= TRACE_TOL
    m, g = pk.misfit_and_gradient(pk.SosMap(grid, z["c0"]), pk.ChannelData(z["obs"], geom, grid.dt),
                                  pulse, damp)
    assert rel_l2(g.values, z["grad"]) <= GRAD_TOL
    g2 = pk.compute_gradient(pk.SosMap(grid, z["c0"]), pk.ChannelData(z["obs"], geom, grid.dt),
                             pulse, damp)
    assert np.array_equal(g.values, g2.values)


@pytest.mark.parametrize("engine", ENGINES)
def test_config0_traces_vs_golden(gpu, golden_dir, engine):
    z = np.load(golden_dir / "config0.npz")
    wl, grid, geom, pulse, damp = config_setup(0)
    assert np.array_equal(wl.c_true[0], z["c_true"])
    eng = _engine(grid, geom, pulse, damp, engine)
    eng.set_model(wl.c_true)
    tr = eng.forward().cpu().numpy()
    assert rel_l2(tr, z["obs_f32"]) <= TRACE_TOL


@pytest.mark.parametrize("engine", ENGINES)
@pytest.mark.parametrize("store", STORES)
def test_config0_gradient_fixed_obs(gpu, golden_dir, engine, store):
    """Fixed float64 observations from the reference (the hard protocol of §7.3-1)."""
    z = np.load(golden_dir / "config0.npz")
    wl, grid, geom, pulse, damp = config_setup(0)
    eng = _engine(grid, geom, pulse, damp, engine)
    eng.set_model(np.full((1, grid.nx, grid.nz), 1540.0))
    obs, _ = oracle.forward_sweep(wl.c_true[0], damp.values, grid.dx, grid.dt, pulse.samples,
                                  geom.tx_nodes(), geom.rx_nodes())
    mis, g = eng.misfit_and_gradient(torch.as_tensor(obs).to(gpu), store=store)
    assert rel_l2(g[0].cpu().numpy(), z["grad"]) <= GRAD_TOL
    assert abs(float(mis[0]) - float(z["misfit"])) <= 1e-4 * float(z["misfit"])


def test_config0_gradient_own_obs(gpu, golden_dir):
    """Observed data simulated by the GPU's own forward (config 0's protocol)."""
    z = np.load(golden_dir / "config0.npz")
    wl, grid, geom, pulse, damp = config_setup(0)
    eng = _engine(grid, geom, pulse, damp, "auto")
    eng.set_model(wl.c_true)
    obs = eng.forward().double()
    eng.set_model(np.full((1, grid.nx, grid.nz), 1540.0))
    _, g = eng.misfit_and_gradient(obs)
    assert rel_l2(g[0].cpu().numpy(), z["grad"]) <= GRAD_TOL


@pytest.mark.parametrize("engine", ("auto", "stepwise"))
def test_variable_density_vs_oracle(gpu, engine):
    wl, grid, geom, pulse, damp = small_linear(rho=True, seed=11)
    rho = wl.rho[0]
    assert rho.min() < 1000.0 or rho.max() > 1000.0
    obs, _ = oracle.forward_sweep(wl.c_true[0], damp.values, grid.dx, grid.dt, pulse.samples,
                                  geom.tx_nodes(), geom.rx_nodes(), rho=rho)
    eng = _engine(grid, geom, pulse, damp, engine, has_rho=True)
    eng.set_model(wl.c_true, rho[None])
    tr = eng.forward().cpu().numpy()
    assert rel_l2(tr, obs) <= TRACE_TOL
    c0 = np.full((grid.nx, grid.nz), 1540.0)
    m_ref, g_ref, _ = oracle.misfit_gradient(c0, damp.values, grid.dx, grid.dt, pulse.samples,
                                             geom.tx_nodes(), geom.rx_nodes(), obs,
                                             element_nodes=geom.element_nodes, rho=rho)
    eng.set_model(c0[None], rho[None])
    for store in STORES:
        mis, g = eng.misfit_and_gradient(torch.as_tensor(obs).to(gpu), store=store)
        assert rel_l2(g[0].cpu().numpy(), g_ref) <= GRAD_TOL
        assert abs(float(mis[0]) - m_ref) <= 1e-4 * m_ref


def test_density_api_constant_rho_equals_plain(gpu):
    wl, grid, geom, pulse, damp = small_linear(seed=5)
    sos = pk.SosMap(grid, wl.c_true[0])
    a = pk.simulate_all(sos, geom, pulse, damp)
    b = pk.simulate_all(sos, geom, pulse, damp, density=np.full(grid.shape, 1000.0))
    # different engines (density runs stepwise with f32 state): agree to storage rounding
    assert rel_l2(b.traces, a.traces) <= 1e-6


def test_batch_of_phantoms_equals_individual(gpu):
    wl, grid, geom, pulse, damp = small_linear(seed=21)
    rng = np.random.default_rng(0)
    cs = [wl.c_true[0], np.full(grid.shape, 1540.0), wl.c_true[0] + rng.uniform(-5, 5, grid.shape)]
    obs_list, single = [], []
    for c in cs:
        obs_list.append(pk.simulate_all(pk.SosMap(grid, c + 3.0), geom, pulse, damp))
    for c, o in zip(cs, obs_list):
        single.append(pk.misfit_and_gradient(pk.SosMap(grid, c), o, pulse, damp))
    ms, gs = pk.misfit_and_gradient_batch([pk.SosMap(grid, c) for c in cs], obs_list, pulse, damp)
    for (m1, g1), m2, g2 in zip(single, ms, gs):
        assert rel_l2(g2.values, g1.values) <= 1e-12
        assert abs(m1 - m2) <= 1e-12 * abs(m1)


def test_duplicate_receivers_accumulate_like_add_at(gpu):
    """np.add.at semantics (adjoint.py:127): a node listed twice receives both residuals."""
    z, grid, geom, pulse, damp = ring48()
    rxp = np.array(geom.rx_pattern)
    rxp[:, 2] = rxp[:, 0]  # duplicate receiver node in every shot
    g2 = pk.AcquisitionGeometry(grid, geom.element_nodes, rxp, 0.028)
    obs, _ = oracle.forward_sweep(z["c_true"], damp.values, grid.dx, grid.dt, pulse.samples,
                                  g2.tx_nodes(), g2.rx_nodes())
    obs[:, 2] += 0.01 * obs[:, 0]  # different obs on the duplicate
    m_ref, g_ref, _ = oracle.misfit_gradient(z["c0"], damp.values, grid.dx, grid.dt,
                                             pulse.samples, g2.tx_nodes(), g2.rx_nodes(), obs,
                                             element_nodes=g2.element_nodes)
    for engine in ENGINES:
        eng = _engine(grid, g2, pulse, damp, engine)
        eng.set_model(z["c0"][None])
        mis, g = eng.misfit_and_gradient(torch.as_tensor(obs).to(gpu))
        assert rel_l2(g[0].cpu().numpy(), g_ref) <= GRAD_TOL
        assert abs(float(mis[0]) - m_ref) <= 1e-4 * m_ref


def test_unmasked_gradient_uses_full_history(gpu):
    z, grid, geom, pulse, damp = ring48()
    m_ref, g_ref, _ = oracle.misfit_gradient(z["c0"], damp.values, grid.dx, grid.dt,
                                             pulse.samples, geom.tx_nodes(), geom.rx_nodes(),
                                             z["obs"], mask=False)
    _, g = pk.misfit_and_gradient(pk.SosMap(grid, z["c0"]), pk.ChannelData(z["obs"], geom, grid.dt),
                                  pulse, damp, mask=False)
    assert rel_l2(g.values, g_ref) <= GRAD_TOL
    assert np.abs(g.values[damp.values > 0]).max() > 0  # PML cells carry gradient when unmasked


def test_zero_residual_gives_zero_gradient(gpu):
    wl, grid, geom, pulse, damp = small_linear(seed=2)
    eng = _engine(grid, geom, pulse, damp, "auto")
    eng.set_model(wl.c_true)
    obs = eng.forward().double()
    mis, g = eng.misfit_and_gradient(obs)
    assert float(mis[0]) == 0.0
    assert float(g.abs().max()) == 0.0


def test_simulate_wavefield_vs_oracle(gpu):
    z, grid, geom, pulse, damp = ring48()
    src = (20, 24)
    f = pk.simulate_wavefield(pk.SosMap(grid, z["c_true"]), pulse, src, damp)
    _, ref = oracle.forward_sweep(z["c_true"], damp.values, grid.dx, grid.dt, pulse.samples,
                                  np.array([src]), None, store=True)
    assert f.shape == (grid.nt, grid.nx, grid.nz)
    assert rel_l2(f, ref[0]) <= TRACE_TOL


def test_errors_match_reference_types(gpu):
    z, grid, geom, pulse, damp = ring48()
    thick = pk.build_pml(grid, 12)  # ring elements now sit in the band
    with pytest.raises(pk.GeometryError):
        pk.simulate_all(pk.SosMap(grid, z["c0"]), geom, pulse, thick)
    fast = pk.SosMap(grid, np.full(grid.shape, 4000.0))
    with pytest.raises(ValueError, match="CFL"):
        pk.simulate_all(fast, geom, pulse, damp)
    big = pk.SourcePulse(np.full(grid.nt, 1e300), grid.dt, 2e5)
    with pytest.raises(pk.NumericError):
        pk.simulate_all(pk.SosMap(grid, z["c0"]), geom, big, damp)


def test_cluster_lap_store_vs_reference(gpu, golden_dir):
    """The cluster engine's L(u)-history store (the forward keeps the imaging
    operand, the adjoint carries only lam): ring48 and config 0 against the
    reference fixtures; box-only like the strips (unmasked gradients refuse it); it is
    the cluster engine's auto store."""
    z, grid, geom, pulse, damp = ring48()
    eng = _engine(grid, geom, pulse, damp, "cluster")
    from paper_2603_04070_b200.engine import STORE_LAP

    assert eng.pick_store(True) == STORE_LAP
    eng.set_model(z["c0"][None])
    obs = torch.as_tensor(z["obs"]).to(gpu)
    mis, g = eng.misfit_and_gradient(obs, store="lap")
    assert eng.last_engine == "cluster"
    assert rel_l2(g[0].cpu().numpy(), z["grad"]) <= GRAD_TOL
    assert abs(float(mis[0]) - float(z["misfit"])) <= 1e-4 * float(z["misfit"])
    with pytest.raises(ValueError, match="mask=True"):
        eng.misfit_and_gradient(obs, store="lap", mask=False)
    _, gs = eng.misfit_and_gradient(obs, store="strips")
    assert rel_l2(g.cpu().numpy(), gs.cpu().numpy()) <= 1e-6
    wl, grid, geom, pulse, damp = config_setup(0)
    zc = np.load(golden_dir / "config0.npz")
    eng = _engine(grid, geom, pulse, damp, "cluster")
    eng.set_model(np.full((1,) + grid.shape, 1540.0))
    obs, _ = oracle.forward_sweep(wl.c_true[0], damp.values, grid.dx, grid.dt, pulse.samples,
                                  geom.tx_nodes(), geom.rx_nodes())
    _, g = eng.misfit_and_gradient(torch.as_tensor(obs).to(gpu), store="lap")
    assert rel_l2(g[0].cpu().numpy(), zc["grad"]) <= GRAD_TOL


@pytest.mark.parametrize("engine", ENGINES)
def test_arith_option_f32_default_f64_precise(gpu, engine):
    """dufwi_geometry_t.arith: the default f32 increment form sits at the f32-storage
    error level (~5e-7 on traces); arith="f64" evaluates the reference's operation
    order in f64 — on the cluster engine the whole sweep, so only the final f32
    rounding of the samples remains (<= 1e-7)."""
    z, grid, geom, pulse, damp = ring48()
    errs = {}
    for arith in ("f32", "f64"):
        eng = fwd.get_engine(grid, geom.tx_nodes(), geom.rx_nodes(), geom.element_nodes,
                             pulse.samples, damp, engine=engine, arith=arith)
        assert eng.arith == arith
        eng.set_model(z["c_true"][None])
        errs[arith] = rel_l2(eng.forward().cpu().numpy(), z["obs"])
        eng.set_model(z["c0"][None])
        mis, g = eng.misfit_and_gradient(torch.as_tensor(z["obs"]).to(gpu))
        assert rel_l2(g[0].cpu().numpy(), z["grad"]) <= GRAD_TOL
    assert errs["f32"] <= 2e-6
    assert errs["f64"] <= (1e-7 if engine == "cluster" else 2e-6)
    if engine == "cluster":
        assert errs["f64"] < errs["f32"]
    with pytest.raises(ValueError, match="arith"):
        fwd.get_engine(grid, geom.tx_nodes(), geom.rx_nodes(), geom.element_nodes,
                       pulse.samples, damp, engine=engine, arith="f16")
