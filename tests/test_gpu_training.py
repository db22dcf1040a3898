"""Training-side physics on the GPU, through libdufwi.

* batched_gradients: B samples as B phantoms of one launch set == the oracle's
  per-sample misfit gradient (adjoint.py:94-138), relative L2 <= 1e-4;
* prepare_block_dataset(k=1): the rolled estimate and its gradient equal the
  oracle restatement of _roll_estimate (unfold.py:145-160) with the same net;
  a sample whose observed data make the physics pass fail is skipped;
* advance_block_dataset == prepare_block_dataset(k+1) (unfold.py:190-197 docstring);
* simulate_dataset == simulate_all per sample (same kernels, bit for bit) and
  == the oracle forward (<= 1e-4), with the FWIR files written.
"""

from __future__ import annotations

import numpy as np
import pytest
import torch

import oracle
import paper_2603_04070_b200 as pk
from paper_2603_04070_b200 import raster
from paper_2603_04070_b200.network import make_update_nets
from paper_2603_04070_b200.training import (advance_block_dataset, batched_gradients,
                                            prepare_block_dataset, simulate_dataset)

from ._cases import rel_l2, small_linear

pytestmark = pytest.mark.gpu


def _samples(n=3, seed=3):
    wl, grid, geom, pulse, damp = small_linear(seed=seed)
    tx, rx = geom.tx_nodes(), geom.rx_nodes()
    rng = np.random.default_rng(11)
    truths, samples = [], []
    for i in range(n):
        c = np.full(grid.shape, 1540.0)
        x0, z0 = rng.integers(16, 36, size=2)
        # contrast 20-40 m/s either sign: a residual of ~1% of the traces, as in config 0
        c[x0 - 4:x0 + 4, z0 - 4:z0 + 4] += rng.choice([-1.0, 1.0]) * rng.uniform(20, 40)
        obs, _ = oracle.forward_sweep(c, damp.values, grid.dx, grid.dt, pulse.samples, tx, rx)
        samples.append((pk.ChannelData(obs, geom, grid.dt), pk.SosMap(grid, c)))
        truths.append(c)
    setup = pk.InversionSetup(pulse, damp, (1300.0, 1700.0), water_speed=1540.0)
    return samples, setup, grid, geom, pulse, damp


def test_batched_gradients_match_oracle(gpu):
    samples, setup, grid, geom, pulse, damp = _samples()
    c = np.stack([np.full(grid.shape, 1540.0) + 5.0 * i for i in range(len(samples))])
    g, ok = batched_gradients(c, samples, setup)
    assert ok.all()
    for i, (m_obs, _) in enumerate(samples):
        _, g_ref, _ = oracle.misfit_gradient(c[i], damp.values, grid.dx, grid.dt, pulse.samples,
                                             geom.tx_nodes(), geom.rx_nodes(), m_obs.traces,
                                             geom.element_nodes)
        assert rel_l2(g[i], g_ref) <= 1e-4
    # batch size does not change the result
    g2, _ = batched_gradients(c, samples, setup, batch=2)
    assert rel_l2(g2, g) <= 1e-12


def test_prepare_and_advance_block_dataset(gpu):
    samples, setup, grid, geom, pulse, damp = _samples()
    net = make_update_nets(1, seed=4, device=gpu)[0]
    ds1 = prepare_block_dataset(1, samples, [net], setup)
    assert ds1.k == 1 and len(ds1) == len(samples)
    tx, rx = geom.tx_nodes(), geom.rx_nodes()
    for i, (m_obs, c_gt) in enumerate(samples):
        c0 = np.full(grid.shape, 1540.0)
        _, g0, _ = oracle.misfit_gradient(c0, damp.values, grid.dx, grid.dt, pulse.samples, tx, rx,
                                          m_obs.traces, geom.element_nodes)
        c1 = np.clip(c0 + net.predict_update(c0, g0), *setup.bounds)
        _, g1, _ = oracle.misfit_gradient(c1, damp.values, grid.dx, grid.dt, pulse.samples, tx, rx,
                                          m_obs.traces, geom.element_nodes)
        assert rel_l2(ds1.c_maps[i], c1) <= 1e-7  # fp32 net on gradients equal to ~1e-7
        assert rel_l2(ds1.gradients[i], g1) <= 1e-4
        assert np.array_equal(ds1.targets[i], c_gt.values)
    ds0 = prepare_block_dataset(0, samples, [], setup)
    ds1b = advance_block_dataset(ds0, net, samples, setup)
    assert ds1b.k == 1
    assert rel_l2(ds1b.c_maps, ds1.c_maps) <= 1e-12
    assert rel_l2(ds1b.gradients, ds1.gradients) <= 1e-9
    with pytest.raises(ValueError):
        prepare_block_dataset(2, samples, [net], setup)


def test_prepare_skips_failing_sample(gpu, caplog):
    samples, setup, grid, geom, pulse, damp = _samples()
    bad = np.array(samples[1][0].traces)
    bad[0, 0, 5] = 1e300  # residual overflows to inf in the adjoint
    samples[1] = (pk.ChannelData(bad, geom, grid.dt), samples[1][1])
    ds = prepare_block_dataset(0, samples, [], setup)
    assert len(ds) == 2
    assert np.array_equal(ds.targets[1], samples[2][1].values)


def test_simulate_dataset_matches_simulate_all(gpu, tmp_path):
    samples, setup, grid, geom, pulse, damp = _samples()
    maps = [s[1] for s in samples]
    cds = simulate_dataset(maps, geom, pulse, damp, out_dir=tmp_path)
    for i, (cd, m) in enumerate(zip(cds, maps)):
        single = pk.simulate_all(m, geom, pulse, damp)
        assert np.array_equal(cd.traces, single.traces)
        ref, _ = oracle.forward_sweep(m.values, damp.values, grid.dx, grid.dt, pulse.samples,
                                      geom.tx_nodes(), geom.rx_nodes())
        assert rel_l2(cd.traces, ref) <= 1e-4
        d = tmp_path / f"sample_{i:06d}"
        assert np.array_equal(raster.read_raster(d / "cd.fwir"), cd.traces)
        assert np.array_equal(raster.read_raster(d / "sos.fwir"), m.values)
