"""DUFWI parity on the GPU (BASELINE config 1): K=5 unfolded iterations on the
config-0 geometry with random-init 4x(3x3, 32 ch) PyTorch update networks.

Protocol: per-iteration gradients are checked on the ORACLE's
(C_k, M_obs) — fixed float64 observations, the hard case — at relative L2
<= 1e-4; the GPU's own end-to-end trajectory (own observations, fp32 nets) must
land within 1e-3 of the oracle's final SoS map."""

from __future__ import annotations

import copy

import numpy as np
import pytest
import torch

import oracle
import paper_2603_04070_b200 as pk
from paper_2603_04070_b200 import forward as fwd
from paper_2603_04070_b200.network import make_update_nets
from paper_2603_04070_b200.unfold import Reconstructor

from ._cases import config_setup, rel_l2

pytestmark = pytest.mark.gpu


def test_config1_dufwi_matches_oracle(gpu):
    wl, grid, geom, pulse, damp = config_setup(1)
    bounds = pk.cfl_safe_bounds(grid, (1300.0, 3200.0))
    tx, rx = geom.tx_nodes(), geom.rx_nodes()
    nets = make_update_nets(5, seed=0, device=gpu)
    nets64 = [copy.deepcopy(n).double().cpu() for n in nets]

    # oracle trajectory: f64 physics + f64 copies of the same networks
    obs, _ = oracle.forward_sweep(wl.c_true[0], damp.values, grid.dx, grid.dt, pulse.samples, tx, rx)
    c0 = np.full(grid.shape, 1540.0)
    upd = [lambda c, g, n=n: n.predict_update(c, g) for n in nets64]
    maps_ref, grads_ref = oracle.unfold_reconstruct(obs, c0, upd, bounds, damp.values, grid.dx,
                                                    grid.dt, pulse.samples, tx, rx, geom.element_nodes)

    eng = fwd.get_engine(grid, tx, rx, geom.element_nodes, pulse.samples, damp)
    obs_dev = torch.as_tensor(obs).to(gpu)
    # (1) per-iteration gradients on the oracle's C_k (C_0 = clamp(c0))
    cks = [np.clip(c0, *bounds)] + maps_ref[:-1]
    for k, ck in enumerate(cks):
        eng.set_model(ck[None])
        _, g = eng.misfit_and_gradient(obs_dev)
        assert rel_l2(g[0].cpu().numpy(), grads_ref[k]) <= 1e-4, k

    # (2) the GPU's own trajectory from its own observations, fp32 networks
    eng.set_model(wl.c_true)
    own_obs = eng.forward().double()
    rec = Reconstructor(eng, nets, bounds)
    maps = rec.reconstruct(own_obs, torch.full((1,) + grid.shape, 1540.0, dtype=torch.float64,
                                               device=gpu))
    final = maps[-1][0].cpu().numpy()
    assert rel_l2(final, maps_ref[-1]) <= 1e-3
    assert rel_l2(final - 1540.0, maps_ref[-1] - 1540.0) <= 1e-3  # the update itself, not just the background


def test_unfold_infer_public_api(gpu):
    wl, grid, geom, pulse, damp = config_setup(1)
    bounds = pk.cfl_safe_bounds(grid, (1300.0, 3200.0))
    obs = pk.simulate_all(pk.SosMap(grid, wl.c_true[0]), geom, pulse, damp)
    nets = make_update_nets(2, seed=1, device=gpu)
    setup = pk.InversionSetup(pulse, damp, bounds)
    out = pk.unfold_infer(obs, pk.homogeneous_map(grid, 1540.0), nets, setup)
    assert len(out) == 2 and all(isinstance(m, pk.SosMap) for m in out)
    assert out[-1].values.min() >= bounds[0] and out[-1].values.max() <= bounds[1]
    # same as the engine-level reconstructor
    eng = fwd.get_engine(grid, geom.tx_nodes(), geom.rx_nodes(), geom.element_nodes, pulse.samples,
                         damp)
    rec = Reconstructor(eng, nets, bounds)
    maps = rec.reconstruct(torch.as_tensor(obs.traces).to(gpu),
                           torch.full((1,) + grid.shape, 1540.0, dtype=torch.float64, device=gpu))
    assert np.array_equal(maps[-1][0].cpu().numpy(), out[-1].values)


def test_unfold_infer_nonfinite_raises(gpu):
    """Deferred non-finite checks still surface as the reference's NumericError."""
    from ._cases import ring48

    z, grid, geom, pulse, damp = ring48()
    obs = pk.ChannelData(z["obs"], geom, grid.dt)
    big = pk.SourcePulse(np.full(grid.nt, 1e300), grid.dt, 2e5)
    nets = make_update_nets(2, seed=1, device=gpu)
    setup = pk.InversionSetup(big, damp, pk.cfl_safe_bounds(grid, (1300.0, 3200.0)))
    with pytest.raises(pk.NumericError):
        pk.unfold_infer(obs, pk.homogeneous_map(grid, 1540.0), nets, setup)


def test_unfold_infer_batch_equals_single_calls(gpu):
    """unfold_infer_batch (B phantoms, one launch set per stage) == B unfold_infer calls.
    The physics is per unit and bit-identical; the fp32 update net may pick other
    cuDNN algorithms for batch 2 than for batch 1 (rounding-level map differences)."""
    from ._cases import small_linear

    wl, grid, geom, pulse, damp = small_linear(seed=5)
    tx, rx = geom.tx_nodes(), geom.rx_nodes()
    obs_list, c0_list = [], []
    for k, dc in enumerate((25.0, -30.0)):
        c = np.full(grid.shape, 1540.0)
        c[18:30, 20 + 4 * k:30 + 4 * k] += dc
        tr, _ = oracle.forward_sweep(c, damp.values, grid.dx, grid.dt, pulse.samples, tx, rx)
        obs_list.append(pk.ChannelData(tr, geom, grid.dt))
        c0_list.append(pk.SosMap(grid, np.full(grid.shape, 1540.0)))
    nets = make_update_nets(2, seed=3, device=gpu)
    setup = pk.InversionSetup(pulse, damp, (1300.0, 1700.0))
    batch = pk.unfold_infer_batch(obs_list, c0_list, nets, setup)
    for b in range(2):
        single = pk.unfold_infer(obs_list[b], c0_list[b], nets, setup)
        for m_b, m_s in zip(batch[b], single):
            assert rel_l2(m_b.values, m_s.values) <= 1e-7


def test_graphed_reconstruct_equals_eager(gpu):
    """The CUDA-graph replay of the K stages gives the same bits as the eager
    launches, follows new inputs, and is re-captured when the engine's
    workspace is reallocated (the captured addresses would be stale)."""
    wl, grid, geom, pulse, damp = config_setup(1)
    bounds = pk.cfl_safe_bounds(grid, (1300.0, 3200.0))
    eng = fwd.get_engine(grid, geom.tx_nodes(), geom.rx_nodes(), geom.element_nodes,
                         pulse.samples, damp)
    nets = make_update_nets(3, seed=1, device=gpu)
    eng.set_model(wl.c_true)
    obs = eng.forward().double()
    c0 = torch.full((1,) + grid.shape, 1540.0, dtype=torch.float64, device=gpu)
    eager = Reconstructor(eng, nets, bounds, graph=False).reconstruct(obs, c0)
    rec = Reconstructor(eng, nets, bounds, graph=True)
    first = rec.reconstruct(obs, c0)  # eager; the graph is captured on the next call
    assert rec._g is None
    assert all(torch.equal(a, b) for a, b in zip(eager, first))
    graphed = rec.reconstruct(obs, c0)
    assert rec._g is not None
    for a, b in zip(eager, graphed):
        assert torch.equal(a, b)
    # new inputs through the same graph
    obs2 = obs * 0.5
    c02 = c0 + 10.0
    e2 = Reconstructor(eng, nets, bounds, graph=False).reconstruct(obs2, c02)
    g2 = rec.reconstruct(obs2, c02)
    assert all(torch.equal(a, b) for a, b in zip(e2, g2))
    assert not torch.equal(g2[-1], graphed[-1])
    # workspace released -> re-captured, still the same bits
    first = rec._g
    eng.release_workspace()
    g3 = rec.reconstruct(obs, c0)
    assert rec._g is not first
    assert all(torch.equal(a, b) for a, b in zip(eager, g3))
    assert rec.replayed_launches > 0
    # the public API's one-round-trip variant: the same maps on the host, from the
    # replay (graph buffers read without clones) and from eager launches
    want = torch.stack(eager).cpu().numpy()
    assert np.array_equal(rec.reconstruct_host(obs, c0), want)
    assert np.array_equal(rec.reconstruct_host(obs, c0), want)
    assert np.array_equal(Reconstructor(eng, nets, bounds, graph=False).reconstruct_host(obs, c0), want)
    want2 = torch.stack(e2).cpu().numpy()
    assert np.array_equal(rec.reconstruct_host(obs2, c02), want2)


def test_stage_device_equals_torch_update_bitwise(gpu):
    """libdufwi's net input / update kernels give the bits of the torch stage
    clamp(c + predict_update_device(c, g), lo, hi) (unfold.py:263-265)."""
    import torch

    from paper_2603_04070_b200.network import make_update_nets

    net = make_update_nets(1, seed=3, device="cuda")[0]
    gen = torch.Generator(device="cuda").manual_seed(0)
    c = 1540.0 + 30.0 * torch.randn((2, 64, 48), dtype=torch.float64, device="cuda", generator=gen)
    g = torch.randn((2, 64, 48), dtype=torch.float64, device="cuda", generator=gen) * 1e-7
    g[1] = 0.0  # all-zero gradient: second channel 0
    lo, hi = 1500.0, 1560.0
    want = torch.clamp(c + net.predict_update_device(c, g), lo, hi)
    got = net.stage_device(c, g, lo, hi)
    assert torch.equal(got, want)
    assert (got == lo).any() and (got == hi).any()
