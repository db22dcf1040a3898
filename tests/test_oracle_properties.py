"""Properties of the float64 oracle that the reference's SPEC states
and that pin the variable-density extension."""

from __future__ import annotations

import numpy as np

import oracle

DX, DT = 1e-4, 2e-8


def _small(n=28, pml=5, nt=140, seed=1, rho=False):
    rng = np.random.default_rng(seed)
    N = n + 2 * pml
    c = 1540.0 + rng.uniform(-30, 30, (N, N))
    d = oracle.pml_damping(N, N, pml, DX)
    t = np.arange(nt) * DT
    f = 1.5e6
    pulse = np.sin(2 * np.pi * f * (t - 2 / f)) * np.exp(-((t - 2 / f) * f) ** 2)
    pulse /= np.abs(pulse).max()
    el = np.stack([pml + 2 + 3 * np.arange(8), np.full(8, pml)], 1)
    tx = el[[1, 4, 6]]
    rx = np.repeat(el[None], 3, axis=0)
    r = None
    if rho:
        r = 1000.0 + rng.uniform(-50, 100, (N, N))
    return c, d, pulse, el, tx, rx, r


def test_lap_rho_reduces_to_reference_laplacian_at_1000():
    u = np.random.default_rng(0).standard_normal((3, 20, 17))
    a = oracle.lap5(u, DX)
    b = oracle.lap_rho(u, np.full((20, 17), 1000.0), DX)
    assert np.array_equal(a, b)
    assert np.array_equal(oracle.lap_rho_T(u, np.full((20, 17), 1000.0), DX), a)


def test_lap_rho_transpose_is_exact_adjoint():
    rng = np.random.default_rng(3)
    rho = 950 + 150 * rng.random((19, 23))
    u = rng.standard_normal((19, 23))
    v = rng.standard_normal((19, 23))
    lhs = np.sum(oracle.lap_rho(u, rho, DX) * v)
    rhs = np.sum(u * oracle.lap_rho_T(v, rho, DX))
    assert abs(lhs - rhs) <= 1e-12 * abs(lhs)


def test_zero_field_is_fixed_point_and_zero_source_gives_zero_traces():
    c, d, pulse, el, tx, rx, _ = _small()
    tr, _ = oracle.forward_sweep(c, d, DX, DT, np.zeros_like(pulse), tx, rx)
    assert not tr.any()


def test_source_linearity_and_shot_additivity():
    c, d, pulse, el, tx, rx, _ = _small(nt=100)
    a, _ = oracle.forward_sweep(c, d, DX, DT, pulse, tx, rx)
    b, _ = oracle.forward_sweep(c, d, DX, DT, 2.5 * pulse, tx, rx)
    assert np.abs(b - 2.5 * a).max() <= 1e-12 * np.abs(a).max()
    obs = a * 1.01
    m_all, g_all, _ = oracle.misfit_gradient(c, d, DX, DT, pulse, tx, rx, obs, el)
    parts = [oracle.misfit_gradient(c, d, DX, DT, pulse, tx[i:i + 1], rx[i:i + 1], obs[i:i + 1], el)
             for i in range(len(tx))]
    g_sum = sum(p[1] for p in parts)
    assert np.linalg.norm(g_sum - g_all) <= 1e-13 * np.linalg.norm(g_all)
    assert abs(sum(p[0] for p in parts) - m_all) <= 1e-13 * m_all


def test_reciprocity():
    c, d, pulse, el, tx, rx, _ = _small(nt=120)
    a, b = el[1], el[6]
    # E L is self-adjoint in the 1/E-weighted inner product: point-to-point
    # reciprocity holds when source and receiver see the same E
    c[a[0], a[1]] = c[b[0], b[1]] = 1540.0
    ab, _ = oracle.forward_sweep(c, d, DX, DT, pulse, a[None], b[None, None])
    ba, _ = oracle.forward_sweep(c, d, DX, DT, pulse, b[None], a[None, None])
    assert np.abs(ab - ba).max() <= 1e-9 * np.abs(ab).max()


def test_gradient_zero_residual_and_linearity():
    c, d, pulse, el, tx, rx, _ = _small(nt=100)
    tr, _ = oracle.forward_sweep(c, d, DX, DT, pulse, tx, rx)
    m0, g0, _ = oracle.misfit_gradient(c, d, DX, DT, pulse, tx, rx, tr, el)
    assert m0 == 0.0 and not g0.any()
    r = np.random.default_rng(2).standard_normal(tr.shape) * 1e-3
    _, g1, _ = oracle.misfit_gradient(c, d, DX, DT, pulse, tx, rx, tr - r, el)
    _, g2, _ = oracle.misfit_gradient(c, d, DX, DT, pulse, tx, rx, tr - 2 * r, el)
    assert np.linalg.norm(g2 - 2 * g1) <= 1e-10 * np.linalg.norm(g1)


def test_variable_density_gradient_matches_finite_differences():
    c, d, pulse, el, tx, rx, rho = _small(n=24, pml=4, nt=90, rho=True)
    obs, _ = oracle.forward_sweep(c + 8.0, d, DX, DT, pulse, tx, rx, rho=rho)
    _, g, _ = oracle.misfit_gradient(c, d, DX, DT, pulse, tx, rx, obs, el, rho=rho)
    cand = np.argwhere(np.abs(g) > 0.2 * np.abs(g).max())[:5]
    fd = oracle.fd_misfit_derivative(c, d, DX, DT, pulse, tx, rx, obs, [tuple(x) for x in cand],
                                     1e-3, rho=rho)
    adj = g[cand[:, 0], cand[:, 1]]
    assert np.max(np.abs(adj - fd) / np.abs(fd)) < 1e-4


def test_variable_density_constant_rho_gradient_equals_reference_form():
    c, d, pulse, el, tx, rx, _ = _small(nt=80)
    obs, _ = oracle.forward_sweep(c + 5.0, d, DX, DT, pulse, tx, rx)
    m1, g1, _ = oracle.misfit_gradient(c, d, DX, DT, pulse, tx, rx, obs, el)
    m2, g2, _ = oracle.misfit_gradient(c, d, DX, DT, pulse, tx, rx, obs, el,
                                       rho=np.full(c.shape, 1000.0))
    assert m1 == m2 and np.array_equal(g1, g2)


def test_guard_mask_rule():
    d = oracle.pml_damping(20, 20, 3, DX)
    keep = oracle.guard_mask(d, np.array([[10, 5]]), 2)
    assert not keep[10, 5] and not keep[12, 5] and keep[13, 5] and not keep[0, 0]
    assert keep[11, 7] and not keep[11, 6]  # d^2 = 1 + 4 = 5 > 4 kept; 1 + 1 = 2 dropped


def test_unfold_reconstruct_clamps_and_uses_updates():
    c, d, pulse, el, tx, rx, _ = _small(nt=80)
    obs, _ = oracle.forward_sweep(c, d, DX, DT, pulse, tx, rx)
    calls = []

    def upd(cm, g):
        calls.append(g.copy())
        return np.full_like(cm, 5000.0)

    maps, grads = oracle.unfold_reconstruct(obs, np.full(c.shape, 1540.0), [upd, upd],
                                            (1300.0, 3200.0), d, DX, DT, pulse, tx, rx, el)
    assert len(maps) == 2 and np.all(maps[-1] == 3200.0) and len(calls) == 2
