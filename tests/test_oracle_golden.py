"""The CPU oracle is pinned to the reference: fixtures in tests/golden/ were produced
by running fwilab itself (oracle/make_golden.py); the restatement must reproduce
them bit for bit."""

from __future__ import annotations

import hashlib
import json

import numpy as np
import pytest

import oracle

from .conftest import GOLDEN


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


def test_ring48_forward_and_gradient_bit_identical():
    z = np.load(GOLDEN / "ring48.npz")
    d = z["damping"]
    assert np.array_equal(oracle.pml_damping(48, 48, 8, float(z["dx"])), d)
    tx = z["nodes"]
    rx = z["nodes"][z["rx_pattern"]]
    tr, _ = oracle.forward_sweep(z["c_true"], d, float(z["dx"]), float(z["dt"]), z["pulse"], tx, rx)
    assert np.array_equal(tr, z["obs"])
    m, g, trial = oracle.misfit_gradient(z["c0"], d, float(z["dx"]), float(z["dt"]), z["pulse"], tx,
                                         rx, z["obs"], element_nodes=z["nodes"])
    assert np.array_equal(trial, z["trial"])
    assert m == float(z["misfit"])
    assert np.array_equal(g, z["grad"])


def test_gradcheck16_matches_reference_and_its_fd_oracle():
    z = np.load(GOLDEN / "gradcheck16.npz")
    tx = z["nodes"]
    rx = z["nodes"][z["rx_pattern"]]
    d = np.zeros((16, 16))
    m, g, _ = oracle.misfit_gradient(z["c0"], d, float(z["dx"]), float(z["dt"]), z["pulse"], tx,
                                     rx, z["obs"], element_nodes=z["nodes"])
    assert m == float(z["misfit"]) and np.array_equal(g, z["grad"])
    cells = [tuple(c) for c in z["cells"][:4]]
    fd = oracle.fd_misfit_derivative(z["c0"], d, float(z["dx"]), float(z["dt"]), z["pulse"], tx,
                                     rx, z["obs"], cells, 1e-3)
    assert np.array_equal(fd, z["fd"][:4])
    rel = np.abs(g[z["cells"][:, 0], z["cells"][:, 1]] - z["fd"]) / np.abs(z["fd"])
    assert rel.max() < 1e-4  # the reference CLI's own tolerance (cli.py:518)


@pytest.mark.slow
def test_config0_reference_hashes():
    """Config-0 observed traces and gradient: sha256 of the f64 arrays from fwilab."""
    from paper_2603_04070_b200 import configs

    meta = json.loads((GOLDEN / "golden_meta.json").read_text())["cases"]["config0"]
    z = np.load(GOLDEN / "config0.npz")
    wl = configs.make_workload(0, seed=0)
    assert np.array_equal(wl.c_true[0], z["c_true"])
    d = z["damping"]
    tx, rx = wl.nodes[wl.tx], wl.nodes[wl.rx]
    obs, _ = oracle.forward_sweep(wl.c_true[0], d, 1e-4, 2e-8, wl.pulse, tx, rx)
    assert _sha(obs) == meta["obs_sha256_f64"]
    m, g, trial = oracle.misfit_gradient(np.full((160, 160), 1540.0), d, 1e-4, 2e-8, wl.pulse, tx,
                                         rx, obs, element_nodes=wl.nodes)
    assert _sha(trial) == meta["trial_sha256_f64"]
    assert _sha(g) == meta["grad_sha256_f64"] and np.array_equal(g, z["grad"])
    assert m == meta["misfit"]


def test_pml_peak_matches_reference_kat():
    meta = json.loads((GOLDEN / "golden_meta.json").read_text())["kats"]
    lam = 1500.0 / 350e3
    assert oracle.pml_axis_profile(188, 20, lam / 8).max() == meta["dmax_paper"]
    assert abs(meta["dmax_paper"] - 1.46e6) / 1.46e6 < 0.05  # PAPER.md:288 quotes 1.46e6
