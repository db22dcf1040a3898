"""Parity at BASELINE.json's stated sizes against the full-size float64 fixtures
of ``oracle/make_golden_large.py`` (C checker with snapshot checkpointing, the
same arithmetic as the NumPy restatement pinned to the reference):

  config 3  560^2, nt 4000, variable density, 2 transmits, fixed f64 (stored
            f32) observations; strips (the default) and full history
  config 4  1088^2, nt 6000, 2 phantoms x 2 transmits, own observations; strips
  config 2  DUFWI K=5 on phantoms 0-1 of the batch, density: per-stage
            gradients along the device's own trajectory and the final maps
  config 3  DUFWI K=3, all 128 transmits, density

Tolerances (north star): relative L2 <= 1e-4 on traces and per-iteration
gradients, <= 1e-3 on the final SoS map.  Plus size-independent properties at
config 4's full size: zero residual -> zero gradient, residual linearity."""

from __future__ import annotations

import hashlib
import json

import numpy as np
import pytest
import torch

import paper_2603_04070_b200 as pk
from paper_2603_04070_b200 import configs
from paper_2603_04070_b200 import forward as fwd
from paper_2603_04070_b200.network import make_update_nets
from paper_2603_04070_b200.unfold import Reconstructor

from ._cases import rel_l2
from .conftest import GOLDEN

pytestmark = pytest.mark.gpu

LARGE = GOLDEN / "large"
META = json.loads((LARGE / "meta.json").read_text())
DEC = META["trace_decimation"]
TOL, MAP_TOL = 1e-4, 1e-3


def _setup(cfg, n_phantoms, shots=None):
    spec = configs.get_config(cfg)
    wl = configs.make_workload(spec, seed=0, n_phantoms=n_phantoms)
    sel = np.arange(len(wl.tx)) if shots is None else np.asarray(shots)
    grid = pk.Grid2D(spec.n, spec.n, spec.dx, spec.dt, spec.nt)
    geom = pk.AcquisitionGeometry(grid, wl.nodes, wl.rx[sel], 0.0, tx_elements=wl.tx[sel])
    damp = pk.build_pml(grid, spec.pml)
    eng = fwd.get_engine(grid, geom.tx_nodes(), geom.rx_nodes(), geom.element_nodes, wl.pulse,
                         damp, n_phantoms=n_phantoms, has_rho=wl.rho is not None)
    return spec, wl, grid, geom, damp, eng


def _need(key):
    if key not in META:
        pytest.fail(f"fixture {key} missing: run oracle/make_golden_large.py")
    return META[key]


def test_config3_full_nt_density_fixed_obs(gpu):
    _need("A_config3_grad")
    z = np.load(LARGE / "config3_grad.npz")
    spec, wl, grid, geom, damp, eng = _setup(3, 1, z["shots"])
    eng.set_model(wl.c_true, wl.rho)
    tr = eng.forward().cpu().numpy()
    assert rel_l2(tr, z["obs_f32"]) <= TOL
    eng.set_model(np.full((1,) + grid.shape, 1540.0), wl.rho)
    obs = torch.as_tensor(z["obs_f32"].astype(np.float64)).to(gpu)
    for store in ("strips", "full"):
        mis, g, trial = eng.misfit_and_gradient(obs, store=store, return_traces=True)
        assert eng.last_engine == "stepwise"
        e_g = rel_l2(g[0].cpu().numpy(), z["grad"])
        print(f"config3 nt=4000 density {store}: grad rel L2 {e_g:.2e}")
        assert e_g <= TOL, store
        assert rel_l2(trial.cpu().numpy()[:, :, ::DEC], z["trial_dec"]) <= TOL
        assert abs(float(mis[0]) - float(z["misfit"])) <= TOL * float(z["misfit"])


def test_config4_full_nt_two_phantoms(gpu):
    _need("B_config4_grad")
    z = np.load(LARGE / "config4_grad.npz")
    spec, wl, grid, geom, damp, eng = _setup(4, 2, z["shots"])
    assert grid.nx == 1088 and grid.nt == 6000
    eng.set_model(wl.c_true)
    own = eng.forward().double()
    o = own.cpu().numpy()[:, :, ::DEC]
    assert rel_l2(o, z["obs_dec"].reshape(o.shape)) <= TOL
    eng.set_model(np.full((2,) + grid.shape, 1540.0))
    mis, g = eng.misfit_and_gradient(own)  # strips (auto)
    for b in range(2):
        e_g = rel_l2(g[b].cpu().numpy(), z["grad"][b])
        print(f"config4 nt=6000 phantom {b}: grad rel L2 {e_g:.2e}")
        assert e_g <= TOL
        assert abs(float(mis[b]) - float(z["misfit"][b])) <= 1e-3 * float(z["misfit"][b])


def test_config4_full_size_properties(gpu):
    spec, wl, grid, geom, damp, eng = _setup(4, 1, [40, 200])
    eng.set_model(wl.c_true)
    tr = eng.forward().double()
    assert torch.isfinite(tr).all() and float(tr.abs().max()) > 0
    eng.set_model(np.full((1,) + grid.shape, 1540.0))
    own = eng.forward().double()
    mis0, g0 = eng.misfit_and_gradient(own)  # zero residual -> zero gradient
    assert float(mis0[0]) == 0.0 and float(g0.abs().max()) == 0.0
    r = tr - own  # linearity in the residual (the adjoint is linear; f32 state only rounds)
    _, g1 = eng.misfit_and_gradient(own - r)
    _, g2 = eng.misfit_and_gradient(own - 2 * r)
    assert rel_l2(g2.cpu().numpy(), 2 * g1.cpu().numpy()) <= 1e-5


def _weights_sha(nets):
    h = hashlib.sha256()
    for n in nets:
        for p in n.parameters():
            h.update(p.detach().cpu().numpy().tobytes())
    return h.hexdigest()


def _dufwi(gpu, cfg, key, name, n_phantoms):
    meta = _need(key)
    z = np.load(LARGE / name)
    spec, wl, grid, geom, damp, eng = _setup(cfg, n_phantoms)
    nets = make_update_nets(spec.k_stages, seed=meta["net_seed"], device=gpu)
    assert _weights_sha(nets) == meta["net_weights_sha256_f32"]
    bounds = tuple(float(v) for v in z["bounds"])
    assert bounds == pk.cfl_safe_bounds(grid, (1300.0, 3200.0))
    eng.set_model(wl.c_true, wl.rho)
    own = eng.forward().double()
    S = geom.n_p
    o = own.cpu().numpy().reshape(n_phantoms, S, geom.n_r, -1)[:, z["obs_dec_shots"], :, ::DEC]
    assert rel_l2(o, z["obs_dec"]) <= TOL
    rec = Reconstructor(eng, nets, bounds, rho=None if wl.rho is None else torch.as_tensor(wl.rho).to(gpu))
    c0 = torch.full((n_phantoms,) + grid.shape, 1540.0, dtype=torch.float64, device=gpu)
    maps, grads = rec.reconstruct(own, c0, keep_gradients=True)
    for b in range(n_phantoms):
        for k in range(spec.k_stages):
            e = rel_l2(grads[k][b].cpu().numpy(), z["grads"][b, k])
            print(f"config{cfg} DUFWI phantom {b} stage {k}: grad rel L2 {e:.2e}")
            assert e <= TOL, (b, k)
        final = maps[-1][b].cpu().numpy()
        assert rel_l2(final, z["maps"][b, -1]) <= MAP_TOL
        assert rel_l2(final - 1540.0, z["maps"][b, -1] - 1540.0) <= MAP_TOL


def test_config2_dufwi_k5_density(gpu):
    _dufwi(gpu, 2, "C_config2_dufwi", "config2_dufwi.npz", 2)


def test_config3_dufwi_k3_density(gpu):
    _dufwi(gpu, 3, "D_config3_dufwi", "config3_dufwi.npz", 1)
