"""ADMM-TV FWI row on CPU, pinned to tests/golden/fwi.npz made
by running the reference (oracle/make_golden_fwi.py):

* the oracle restatement (oracle/fwi_oracle.py) reproduces the reference's
  tv_prox, lbfgs_minimize and a 3x3 admm_fwi run on ring48 bit for bit;
* the product's tv_prox is bit-exact and its L-BFGS matches to dot-product rounding;
* the batched L-BFGS keeps per-phantom semantics: B problems at once (one of them
  concave, so its curvature pairs are always skipped) equal B separate runs.
"""

from __future__ import annotations

import numpy as np
import pytest
import torch

from oracle import fwi_oracle as fo
from paper_2603_04070_b200 import fwi

from ._cases import ring48
from .conftest import GOLDEN


@pytest.fixture(scope="module")
def z():
    return np.load(GOLDEN / "fwi.npz")


def _quad(A, b):
    def f(x):
        xf = x.ravel()
        return float(0.5 * xf @ A @ xf - b @ xf), (A @ xf - b).reshape(x.shape)
    return f


def test_oracle_tv_prox_and_lbfgs_bit_exact(z):
    out = fo.tv_prox(z["tv_in"], float(z["tv_weight"]), iters=20)
    assert np.array_equal(out, z["tv_out"])
    assert fo.total_variation(out) == float(z["tv_value"])
    x, vals = fo.lbfgs_minimize(_quad(z["quad_A"], z["quad_b"]), z["lb_x0"], iters=7, lr=0.8,
                                memory=3, project=lambda x: np.clip(x, -0.5, 0.5))
    assert np.array_equal(x, z["lb_x"]) and np.array_equal(np.array(vals), z["lb_values"])


def test_oracle_admm_bit_exact(z):
    r, grid, geom, pulse, damp = ring48()
    c, log = fo.admm_fwi(r["obs"], np.full(grid.shape, 1500.0), damp.values, grid.dx, grid.dt,
                         pulse.samples, geom.tx_nodes(), geom.rx_nodes(), geom.element_nodes,
                         int(z["admm_outer"]), int(z["admm_inner"]))
    assert np.array_equal(c, z["admm_map"])
    assert np.array_equal(np.array(log), z["admm_log"])


def test_product_tv_prox_bit_exact(z):
    out = fwi.tv_prox(z["tv_in"], float(z["tv_weight"]), iters=20)
    assert np.array_equal(out, z["tv_out"])
    assert fwi.total_variation(out) == pytest.approx(float(z["tv_value"]), rel=1e-14)
    assert np.array_equal(fwi.tv_prox(z["tv_in"], 0.0), z["tv_in"])
    with pytest.raises(ValueError):
        fwi.tv_prox(z["tv_in"], -1.0)


def test_product_lbfgs_matches_reference(z):
    x, vals = fwi.lbfgs_minimize(_quad(z["quad_A"], z["quad_b"]), z["lb_x0"], iters=7, lr=0.8,
                                 memory=3, project=lambda x: np.clip(x, -0.5, 0.5))
    assert np.max(np.abs(x - z["lb_x"])) <= 1e-12
    assert np.allclose(vals, z["lb_values"], rtol=1e-12, atol=1e-14)


def test_batched_lbfgs_per_phantom_semantics():
    rng = np.random.default_rng(5)
    n = 20
    probs = []
    for k in range(3):
        M = rng.standard_normal((n, n))
        A = M @ M.T / n + np.eye(n)
        if k == 1:
            A = -A  # concave: s.y < 0 always, no pair is ever accepted
        probs.append((A, rng.standard_normal(n)))
    x0 = rng.standard_normal((3, 4, 5))

    def fb(xb):
        fs, gs = [], []
        for (A, b), x in zip(probs, xb.numpy()):
            f, g = _quad(A, b)(x)
            fs.append(f)
            gs.append(g)
        return torch.tensor(fs, dtype=torch.float64), torch.as_tensor(np.stack(gs))

    xb, vb = fwi.lbfgs_minimize_batch(fb, torch.as_tensor(x0), iters=9, lr=0.5, memory=2)
    for k, (A, b) in enumerate(probs):
        xk, vk = fo.lbfgs_minimize(_quad(A, b), x0[k], iters=9, lr=0.5, memory=2)
        assert np.max(np.abs(xb[k].numpy() - xk)) <= 1e-10 * max(1.0, np.abs(xk).max())
        assert np.allclose([float(v[k]) for v in vb], vk, rtol=1e-10, atol=1e-12)


def test_fwi_config_validation():
    fwi.FwiConfig()
    for kw in ({"outer_iters": 0}, {"inner_lbfgs_iters": 0}, {"tv_weight": -1.0},
               {"rho_admm": 0.0}, {"bounds": (2.0, 1.0)}):
        with pytest.raises(ValueError):
            fwi.FwiConfig(**kw)
    e = fwi.FwiDivergenceError(3)
    assert e.outer_iteration == 3 and "outer iteration 3" in str(e)
