"""CPU restatement of the reference's ADMM-TV FWI baseline (fwi.py) — TEST
INFRASTRUCTURE, used only by tests/ as the checker of
``paper_2603_04070_b200.fwi``.

Follows, operation for operation:
* ``_grad_x``/``_grad_z``/``_div``/``total_variation``/``tv_prox`` — fwi.py:70-117
* ``lbfgs_minimize`` (two-loop recursion, fixed step, first step scaled by
  min(1, 1/||g||_1), pairs with s.y <= 1e-12 skipped)                    — fwi.py:120-183
* ``admm_fwi`` (scaled-dual ADMM, default rho = 1e-2 misfit0/||C0||^2,
  tv weight = rho)                                                      — fwi.py:191-248
with the data term from :func:`oracle.misfit_gradient` (itself bit-identical
to fwilab.adjoint.misfit_and_gradient).  Pinned against the
reference by tests/golden/fwi.npz (oracle/make_golden_fwi.py).
"""

from __future__ import annotations

import numpy as np

from .dufwi_oracle import misfit_gradient


def grad_x(v):
    return v[1:, :] - v[:-1, :]


def grad_z(v):
    return v[:, 1:] - v[:, :-1]


def div(zx, zz, shape):
    out = np.zeros(shape)
    out[:-1, :] -= zx
    out[1:, :] += zx
    out[:, :-1] -= zz
    out[:, 1:] += zz
    return out


def total_variation(v) -> float:
    return float(np.abs(grad_x(v)).sum() + np.abs(grad_z(v)).sum())


def tv_prox(v, weight, iters=20):
    v = np.asarray(v, dtype=np.float64)
    if weight == 0.0:
        return v.copy()
    zx = np.zeros((v.shape[0] - 1, v.shape[1]))
    zz = np.zeros((v.shape[0], v.shape[1] - 1))
    for _ in range(iters):
        x = v - weight * div(zx, zz, v.shape)
        zx = np.clip(zx + grad_x(x) / (8.0 * weight), -1.0, 1.0)
        zz = np.clip(zz + grad_z(x) / (8.0 * weight), -1.0, 1.0)
    return v - weight * div(zx, zz, v.shape)


def lbfgs_minimize(value_grad_fn, x0, iters, lr, memory=5, project=None):
    x = np.array(x0, dtype=np.float64)
    s_list, y_list, values = [], [], []
    f, g = value_grad_fn(x)
    values.append(f)
    for it in range(iters):
        if not np.isfinite(f) or not np.all(np.isfinite(g)):
            raise FloatingPointError(f"non-finite objective at inner step {it}")
        if s_list:
            q = g.ravel().copy()
            alphas, rhos = [], []
            for s, y in zip(reversed(s_list), reversed(y_list)):
                rho = 1.0 / float(y.ravel() @ s.ravel())
                alpha = rho * float(s.ravel() @ q)
                q -= alpha * y.ravel()
                alphas.append(alpha)
                rhos.append(rho)
            s_last, y_last = s_list[-1], y_list[-1]
            gamma = float(s_last.ravel() @ y_last.ravel()) / float(y_last.ravel() @ y_last.ravel())
            r = gamma * q
            for (s, y), alpha, rho in zip(zip(s_list, y_list), reversed(alphas), reversed(rhos)):
                beta = rho * float(y.ravel() @ r)
                r += (alpha - beta) * s.ravel()
            direction = -r.reshape(x.shape)
        else:
            g1 = float(np.abs(g).sum())
            direction = -g * (min(1.0, 1.0 / g1) if g1 > 0 else 1.0)
        x_new = x + lr * direction
        if project is not None:
            x_new = project(x_new)
        f_new, g_new = value_grad_fn(x_new)
        s = x_new - x
        y = g_new - g
        if float(y.ravel() @ s.ravel()) > 1e-12:
            s_list.append(s)
            y_list.append(y)
            if len(s_list) > memory:
                s_list.pop(0)
                y_list.pop(0)
        x, f, g = x_new, f_new, g_new
        values.append(f)
    return x, values


def admm_fwi(obs, c0, d, dx, dt, pulse, tx, rx, element_nodes, outer_iters, inner_iters,
             inner_lr=1.0, tv_weight=None, rho_admm=None, bounds=(1300.0, 3200.0)):
    """Returns (final map, misfit log) like fwi.admm_fwi."""
    c_min, c_max = bounds
    c = np.array(c0, dtype=np.float64)

    def fidelity(values):
        mis, g, _ = misfit_gradient(values, d, dx, dt, pulse, tx, rx, obs, element_nodes)
        return mis, g

    misfit0, _ = fidelity(c)
    rho = rho_admm if rho_admm is not None else 1e-2 * misfit0 / float(np.sum(c * c))
    lam = tv_weight if tv_weight is not None else rho
    z = c.copy()
    w = np.zeros_like(c)
    log = [misfit0]
    for _ in range(outer_iters):
        def augmented(values):
            mis, grad = fidelity(values)
            diff = values - z + w
            return mis + 0.5 * rho * float(np.sum(diff * diff)), grad + rho * diff

        c, _ = lbfgs_minimize(augmented, c, iters=inner_iters, lr=inner_lr,
                              project=lambda x: np.clip(x, c_min, c_max))
        c = np.clip(c, c_min, c_max)
        z = tv_prox(c + w, lam / rho)
        w = w + c - z
        mis, _ = fidelity(c)
        log.append(mis)
    return c, log
