"""TEST INFRASTRUCTURE — float64 NumPy restatement of the reference's physics step.

This is the checker the CUDA path is compared against; it is never called by the
product package.  Every function cites the reference code it restates
(paths relative to ``/root/reference/pkg/src/fwilab``).  Operation order inside
each update follows the reference exactly, so on the reference's own geometry the
results are bit-identical (pinned by ``tests/test_oracle_golden.py`` against
fixtures produced by ``oracle/make_golden.py`` from the real package).

Extensions beyond the reference (all reduce to it exactly when unused):

* general transmit/receive node lists ``tx (P,2)`` / ``rx (P,R,2)`` so a
  transmit subset of a linear array can be expressed;
* variable density ``rho``: ``L_rho u = rho div(1/rho grad u)``
  with face inverse-density the mean of the two cell inverse densities, and its
  exact discrete transpose for the adjoint.  ``parity unpinned`` by the
  reference for rho != const; pinned by constant-rho reduction (bit-exact for
  rho = 1000) and a finite-difference gradient check.
"""

from __future__ import annotations

import math

import numpy as np

__all__ = [
    "pml_axis_profile",
    "pml_damping",
    "step_coeffs",
    "lap5",
    "rho_face_weights",
    "lap_rho",
    "lap_rho_T",
    "forward_sweep",
    "misfit_gradient",
    "guard_mask",
    "fd_misfit_derivative",
    "unfold_reconstruct",
    "ORACLE_PML_C_REF",
]

#: damping calibration speed, forward.py:47-48
ORACLE_PML_C_REF = 1500.0


# --------------------------------------------------------------------------- PML
def pml_axis_profile(n: int, thickness: int, dx: float,
                     target_attenuation: float = 1e-3, exponent: float = 2.0) -> np.ndarray:
    """1-D damping ramp along one axis (forward.py:113-118 and :129-133)."""
    if thickness == 0:
        return np.zeros(n)
    peak = (-math.log(target_attenuation) * ORACLE_PML_C_REF * (exponent + 1.0)
            / (2.0 * thickness * dx))
    i = np.arange(n)
    edge_dist = np.minimum(i, n - 1 - i).astype(np.float64)
    frac = np.clip((thickness - edge_dist) / thickness, 0.0, None)
    return peak * frac ** exponent


def pml_damping(nx: int, nz: int, thickness: int, dx: float,
                target_attenuation: float = 1e-3, exponent: float = 2.0) -> np.ndarray:
    """(nx, nz) damping map; corners take the max of the axis ramps (forward.py:135-137)."""
    px = pml_axis_profile(nx, thickness, dx, target_attenuation, exponent)
    pz = pml_axis_profile(nz, thickness, dx, target_attenuation, exponent)
    return np.maximum(px[:, None], pz[None, :])


def step_coeffs(c: np.ndarray, d: np.ndarray, dt: float):
    """A, B, E of the explicit damped update (forward.py:226-234)."""
    ddt = d * dt
    den = 1.0 + ddt
    return (2.0 - ddt ** 2) / den, (ddt - 1.0) / den, c ** 2 * dt * dt / den


# --------------------------------------------------------------------- operators
def lap5(u: np.ndarray, dx: float) -> np.ndarray:
    """5-point Laplacian, zero outside, on the last two axes (forward.py:211-223).

    Accumulation order (x-1, x+1, z-1, z+1 after -4u) matches the reference so
    float64 results are bit-identical.
    """
    acc = -4.0 * u
    acc[..., 1:, :] += u[..., :-1, :]
    acc[..., :-1, :] += u[..., 1:, :]
    acc[..., :, 1:] += u[..., :, :-1]
    acc[..., :, :-1] += u[..., :, 1:]
    acc /= dx * dx
    return acc


def rho_face_weights(rho: np.ndarray):
    """Per-cell face weights w = rho_i * (q_i + q_j)/2, q = 1/rho (G3 extension).

    Returns (w_xm, w_xp, w_zm, w_zp, W) with W the face-weight sum in that order.
    Faces on the outer edge use q_j := q_i.  For constant rho every weight is
    rho*(1/rho), exactly 1.0 for rho = 1000, so ``lap_rho`` reduces to ``lap5``.
    """
    q = 1.0 / rho
    qxm = q.copy(); qxm[1:, :] = q[:-1, :]
    qxp = q.copy(); qxp[:-1, :] = q[1:, :]
    qzm = q.copy(); qzm[:, 1:] = q[:, :-1]
    qzp = q.copy(); qzp[:, :-1] = q[:, 1:]
    w_xm = rho * (0.5 * (q + qxm))
    w_xp = rho * (0.5 * (q + qxp))
    w_zm = rho * (0.5 * (q + qzm))
    w_zp = rho * (0.5 * (q + qzp))
    wsum = ((w_xm + w_xp) + w_zm) + w_zp
    return w_xm, w_xp, w_zm, w_zp, wsum


def lap_rho(u: np.ndarray, rho: np.ndarray, dx: float, weights=None) -> np.ndarray:
    """rho * div(1/rho grad u), zero outside the grid (G3 extension)."""
    w_xm, w_xp, w_zm, w_zp, wsum = weights if weights is not None else rho_face_weights(rho)
    acc = -wsum * u
    acc[..., 1:, :] += w_xm[1:, :] * u[..., :-1, :]
    acc[..., :-1, :] += w_xp[:-1, :] * u[..., 1:, :]
    acc[..., :, 1:] += w_zm[:, 1:] * u[..., :, :-1]
    acc[..., :, :-1] += w_zp[:, :-1] * u[..., :, 1:]
    acc /= dx * dx
    return acc


def lap_rho_T(v: np.ndarray, rho: np.ndarray, dx: float, weights=None) -> np.ndarray:
    """Exact transpose of :func:`lap_rho`: neighbour j contributes w_{j->i} v_j."""
    w_xm, w_xp, w_zm, w_zp, wsum = weights if weights is not None else rho_face_weights(rho)
    acc = -wsum * v
    acc[..., 1:, :] += w_xp[:-1, :] * v[..., :-1, :]
    acc[..., :-1, :] += w_xm[1:, :] * v[..., 1:, :]
    acc[..., :, 1:] += w_zp[:, :-1] * v[..., :, :-1]
    acc[..., :, :-1] += w_zm[:, 1:] * v[..., :, 1:]
    acc /= dx * dx
    return acc


def _ops(rho, dx):
    if rho is None:
        return (lambda u: lap5(u, dx)), (lambda v: lap5(v, dx))
    w = rho_face_weights(np.asarray(rho, dtype=np.float64))
    return (lambda u: lap_rho(u, rho, dx, w)), (lambda v: lap_rho_T(v, rho, dx, w))


# ------------------------------------------------------------------------ sweeps
def forward_sweep(c, d, dx, dt, pulse, tx, rx=None, store=False, rho=None):
    """All transmissions stepped together (forward.py:273-313).

    ``tx`` (P,2) int; ``rx`` (P,R,2) int or None.  Per step: update, inject the
    source at the transmit node, sample receivers, store (the reference order).
    Returns (traces (P,R,nt) | None, fields (P,nt,nx,nz) | None).
    """
    c = np.asarray(c, dtype=np.float64)
    d = np.asarray(d, dtype=np.float64)
    pulse = np.asarray(pulse, dtype=np.float64)
    tx = np.asarray(tx, dtype=np.int64)
    nt = pulse.shape[0]
    n_p = tx.shape[0]
    A, B, E = step_coeffs(c, d, dt)
    L, _ = _ops(rho, dx)
    prev = np.zeros((n_p,) + c.shape)
    prev2 = np.zeros_like(prev)
    shots = np.arange(n_p)
    traces = None if rx is None else np.empty((n_p, rx.shape[1], nt))
    fields = np.empty((n_p, nt) + c.shape) if store else None
    for t in range(nt):
        cur = A * prev + B * prev2 + E * L(prev)
        cur[shots, tx[:, 0], tx[:, 1]] += pulse[t]
        if traces is not None:
            traces[:, :, t] = cur[shots[:, None], rx[:, :, 0], rx[:, :, 1]]
        if fields is not None:
            fields[:, t] = cur
        prev2, prev = prev, cur
    if traces is not None and not np.all(np.isfinite(traces)):
        raise FloatingPointError("simulation diverged: non-finite receiver samples")
    return traces, fields


def guard_mask(d, element_nodes, guard_radius=2):
    """Cells kept in the gradient: undamped and farther than ``guard_radius``
    from every element node (adjoint.py:75-91)."""
    keep = np.asarray(d) == 0.0
    ix = np.arange(keep.shape[0])[:, None]
    iz = np.arange(keep.shape[1])[None, :]
    for nx_, nz_ in np.asarray(element_nodes):
        keep &= (ix - nx_) ** 2 + (iz - nz_) ** 2 > guard_radius ** 2
    return keep


def misfit_gradient(c, d, dx, dt, pulse, tx, rx, obs, element_nodes=None,
                    mask=True, guard_radius=2, rho=None):
    """Misfit and adjoint-state SoS gradient (adjoint.py:94-138), general tx/rx.

    Reverse sweep per step: lam = A lam1 + L^T(E lam1) + B lam2, residual added
    at receiver nodes with duplicates accumulating, then for t >= 1 the imaging
    term dE/dc * sum_p L(u_p[t-1]) lam_p[t]; mask applied after accumulation.
    """
    c = np.asarray(c, dtype=np.float64)
    d = np.asarray(d, dtype=np.float64)
    rx = np.asarray(rx, dtype=np.int64)
    traces, fields = forward_sweep(c, d, dx, dt, pulse, tx, rx, store=True, rho=rho)
    diff = traces - np.asarray(obs, dtype=np.float64)
    resid = 2.0 * diff
    misfit = float(np.sum(diff ** 2))
    A, B, E = step_coeffs(c, d, dt)
    dEdc = 2.0 * c * dt ** 2 / (1.0 + d * dt)
    L, LT = _ops(rho, dx)
    n_p = rx.shape[0]
    shot_col = np.arange(n_p)[:, None]
    lam_next = np.zeros((n_p,) + c.shape)
    lam_next2 = np.zeros_like(lam_next)
    grad = np.zeros(c.shape)
    for t in range(pulse.shape[0] - 1, -1, -1):
        lam = A * lam_next + LT(E * lam_next) + B * lam_next2
        np.add.at(lam, (shot_col, rx[:, :, 0], rx[:, :, 1]), resid[:, :, t])
        if t >= 1:
            grad += dEdc * np.einsum("pij,pij->ij", L(fields[:, t - 1]), lam)
        lam_next2, lam_next = lam_next, lam
    if not np.all(np.isfinite(grad)):
        raise FloatingPointError("gradient blow-up")
    if mask:
        nodes = element_nodes if element_nodes is not None else np.concatenate(
            [np.asarray(tx).reshape(-1, 2), rx.reshape(-1, 2)])
        grad = np.where(guard_mask(d, nodes, guard_radius), grad, 0.0)
    return misfit, grad, traces


def fd_misfit_derivative(c, d, dx, dt, pulse, tx, rx, obs, cells, eps, rho=None):
    """Central-difference misfit derivative at selected cells (adjoint.py:154-186)."""
    out = np.empty(len(cells))
    base = np.array(c, dtype=np.float64)
    for k, (i, j) in enumerate(cells):
        vals = []
        for sgn in (1.0, -1.0):
            pert = base.copy()
            pert[i, j] += sgn * eps
            tr, _ = forward_sweep(pert, d, dx, dt, pulse, tx, rx, rho=rho)
            vals.append(float(np.sum((np.asarray(obs) - tr) ** 2)))
        out[k] = (vals[0] - vals[1]) / (2.0 * eps)
    return out


def unfold_reconstruct(obs, c0, predict_updates, bounds, d, dx, dt, pulse, tx, rx,
                       element_nodes=None, rho=None, guard_radius=2):
    """K-stage unfolded inference (unfold.py:253-267 with clamp_sos :134-142).

    ``predict_updates`` is a list of callables (c, g) -> update in m/s.
    Returns the list of estimates and the per-stage gradients.
    """
    lo, hi = bounds
    c = np.clip(np.asarray(c0, dtype=np.float64), lo, hi)
    maps, grads = [], []
    for f in predict_updates:
        _, g, _ = misfit_gradient(c, d, dx, dt, pulse, tx, rx, obs, element_nodes,
                                  rho=rho, guard_radius=guard_radius)
        grads.append(g)
        c = np.clip(c + f(c, g), lo, hi)
        maps.append(c)
    return maps, grads
