"""The C float64 checker (oracle/dufwi_oracle_c.c) is pinned to the NumPy
restatement (itself pinned bit-for-bit to the reference by test_oracle_golden):
traces and misfits bit-identical, gradients to rounding (shot-summation order),
snapshot checkpointing bit-identical to any other segment length."""

from __future__ import annotations

import json

import numpy as np
import pytest

import oracle
from oracle import c_oracle as co

from ._cases import rel_l2, small_linear
from .conftest import GOLDEN


@pytest.fixture(scope="module", autouse=True)
def _built():
    co.build()


def test_ring48_matches_reference_fixture():
    z = np.load(GOLDEN / "ring48.npz")
    tx = z["nodes"]
    rx = z["nodes"][z["rx_pattern"]]
    m, g, tr = co.misfit_gradient(z["c0"], z["damping"], float(z["dx"]), float(z["dt"]), z["pulse"],
                                  tx, rx, z["obs"], element_nodes=z["nodes"], threads=3)
    assert np.array_equal(tr, z["trial"])  # fwilab's own simulate_all, bit for bit
    assert m == float(z["misfit"])
    assert rel_l2(g, z["grad"]) < 1e-13


@pytest.mark.parametrize("rho", [False, True])
def test_matches_numpy_oracle_and_segments(rho):
    wl, grid, geom, pulse, damp = small_linear(rho=rho, nt=240)
    tx, rx = geom.tx_nodes(), geom.rx_nodes()
    r = wl.rho[0] if rho else None
    obs, _ = oracle.forward_sweep(wl.c_true[0], damp.values, grid.dx, grid.dt, wl.pulse, tx, rx,
                                  rho=r)
    obs_c, _ = co.forward_sweep(wl.c_true[0], damp.values, grid.dx, grid.dt, wl.pulse, tx, rx,
                                rho=r, threads=2)
    assert np.array_equal(obs, obs_c)
    c0 = np.full(grid.shape, 1540.0)
    m1, g1, t1 = oracle.misfit_gradient(c0, damp.values, grid.dx, grid.dt, wl.pulse, tx, rx, obs,
                                        geom.element_nodes, rho=r)
    outs = [co.misfit_gradient(c0, damp.values, grid.dx, grid.dt, wl.pulse, tx, rx, obs,
                               geom.element_nodes, rho=r, seg=seg, threads=th)
            for seg, th in ((2, 1), (13, 3), (240, 2), (None, 8))]
    for m2, g2, t2 in outs:
        assert np.array_equal(t1, t2) and m1 == m2
        assert rel_l2(g2, g1) < 1e-13
        # checkpointing and thread count do not change a single bit
        assert np.array_equal(g2, outs[0][1])


def test_large_fixture_metadata():
    """The full-size fixtures (oracle/make_golden_large.py) are present and consistent."""
    d = GOLDEN / "large"
    meta = json.loads((d / "meta.json").read_text())
    z = np.load(d / "config3_grad.npz")
    assert z["obs_f32"].shape == (2, 256, 4000) and z["grad"].shape == (560, 560)
    assert meta["A_config3_grad"]["nt"] == 4000
    if "B_config4_grad" in meta:
        z = np.load(d / "config4_grad.npz")
        assert z["grad"].shape == (2, 1088, 1088) and z["misfit"].shape == (2,)
    for key, name, shape in (("C_config2_dufwi", "config2_dufwi.npz", (2, 5, 296, 296)),
                             ("D_config3_dufwi", "config3_dufwi.npz", (1, 3, 560, 560))):
        if key in meta:
            z = np.load(d / name)
            assert z["grads"].shape == shape and z["maps"].shape == shape
