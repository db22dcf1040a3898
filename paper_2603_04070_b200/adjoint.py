"""Misfit and adjoint-state gradient API (mirror of ``fwilab.adjoint``).

The gradient is the exact discrete adjoint of the explicit recursion
(adjoint.py:1-19 of the reference):

    lam[t] = r[t] + A lam[t+1] + lap(E lam[t+1]) + B lam[t+2]
    g      = dE/dc * sum_t sum_p lap(u_p[t-1]) * lam_p[t]

computed by ``libdufwi.so``: forward sweep with wavefield history (full f32
history or 1-cell boundary strips + backward reconstruction), residual
kernel, reverse sweep with fused imaging, masked epilogue.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .forward import (DampingProfile, NumericError, SourcePulse, _check_simulation_inputs,
                      _density_values, get_engine, zero_damping)
from .grid import ChannelData, Grid2D, SosMap

__all__ = ["GradientMap", "data_misfit", "gradient_mask", "misfit_and_gradient",
           "compute_gradient", "misfit_and_gradient_batch", "fd_gradient_oracle"]


@dataclass(frozen=True)
class GradientMap:
    """Misfit derivative per cell (adjoint.py:49-64)."""

    grid: Grid2D
    values: np.ndarray

    def __post_init__(self):
        v = np.asarray(self.values, dtype=np.float64)
        if v.shape != self.grid.shape:
            raise ValueError(f"gradient shape {v.shape} != grid {self.grid.shape}")
        if not np.isfinite(v).all():
            raise NumericError("gradient contains non-finite values")
        v = np.ascontiguousarray(v)
        v.flags.writeable = False
        object.__setattr__(self, "values", v)


def data_misfit(m_obs: ChannelData, m_sim: ChannelData) -> float:
    """sum((obs - sim)^2) over all samples (adjoint.py:67-72); host-side utility."""
    if m_obs.shape != m_sim.shape:
        raise ValueError(f"shape mismatch: {m_obs.shape} vs {m_sim.shape}")
    d = m_obs.traces - m_sim.traces
    return float(np.sum(d * d))


def gradient_mask(geometry, damping: DampingProfile, guard_radius: int = 2) -> np.ndarray:
    """Cells kept: undamped and outside every element's guard disk (adjoint.py:75-91).

    The device epilogue applies the same rule in ``finalize_kernel``.
    """
    grid = damping.grid
    keep = damping.values == 0.0
    ix = np.arange(grid.nx)[:, None]
    iz = np.arange(grid.nz)[None, :]
    r2 = guard_radius ** 2
    for x0, z0 in geometry.element_nodes:
        keep &= (ix - x0) ** 2 + (iz - z0) ** 2 > r2
    return keep


def misfit_and_gradient(sos: SosMap, m_obs: ChannelData, pulse: SourcePulse,
                        damping: DampingProfile | None = None, mask: bool = True,
                        guard_radius: int = 2, *, density=None,
                        store: str = "auto", arith: str = "f32") -> tuple[float, GradientMap]:
    """Misfit and its adjoint-state gradient in one forward pass (adjoint.py:94-138).

    ``arith``: "f32" (default) or "f64" — the arithmetic of the sweep kernels
    (include/dufwi.h DUFWI_ARITH_*); "f64" evaluates the reference's operation
    order in float64."""
    import torch

    geometry = m_obs.geometry
    damping = damping if damping is not None else zero_damping(sos.grid)
    _check_simulation_inputs(sos, geometry, pulse, damping)
    rho = _density_values(density, sos.grid)
    eng = get_engine(sos.grid, geometry.tx_nodes(), geometry.rx_nodes(), geometry.element_nodes,
                     pulse.samples, damping, has_rho=rho is not None, arith=arith)
    eng.set_model(sos.values[None], None if rho is None else rho[None])
    obs = torch.as_tensor(m_obs.traces, dtype=torch.float64).to(eng.device)
    try:
        misfit, grad = eng.misfit_and_gradient(obs, mask=mask, guard_radius=guard_radius,
                                               store=store, units=(0, eng.n_units))
    except FloatingPointError as exc:
        raise NumericError(str(exc)) from exc
    return float(misfit[0].item()), GradientMap(sos.grid, grad[0].cpu().numpy())


def compute_gradient(sos: SosMap, m_obs: ChannelData, pulse: SourcePulse,
                     damping: DampingProfile | None = None, mask: bool = True,
                     guard_radius: int = 2, *, density=None, arith: str = "f32") -> GradientMap:
    """Adjoint-state gradient of :func:`data_misfit` (adjoint.py:141-151)."""
    return misfit_and_gradient(sos, m_obs, pulse, damping, mask, guard_radius, density=density,
                               arith=arith)[1]


def misfit_and_gradient_batch(sos_list, obs_list, pulse: SourcePulse,
                              damping: DampingProfile | None = None, mask: bool = True,
                              guard_radius: int = 2, *, density_list=None, arith: str = "f32"):
    """Batched extension: B phantoms sharing one acquisition, one engine launch set.

    Under torch.distributed the (phantom, shot) units are sharded across ranks
    and combined with one all_reduce.
    """
    import torch

    if len(sos_list) != len(obs_list) or not sos_list:
        raise ValueError("need one observed data set per speed map")
    geometry = obs_list[0].geometry
    grid = sos_list[0].grid
    damping = damping if damping is not None else zero_damping(grid)
    for s, o in zip(sos_list, obs_list):
        if not o.geometry.same_acquisition(geometry):
            raise ValueError("batched gradients need one acquisition geometry")
        _check_simulation_inputs(s, o.geometry, pulse, damping)
    if density_list is not None and len(density_list) != len(sos_list):
        raise ValueError("need one density map per speed map")
    B = len(sos_list)
    rho = None
    if density_list is not None:
        rho = np.stack([_density_values(d, grid) for d in density_list])
    eng = get_engine(grid, geometry.tx_nodes(), geometry.rx_nodes(), geometry.element_nodes,
                     pulse.samples, damping, n_phantoms=B, has_rho=rho is not None, arith=arith)
    eng.set_model(np.stack([s.values for s in sos_list]), rho)
    obs = torch.as_tensor(np.concatenate([o.traces for o in obs_list]), dtype=torch.float64)
    try:
        misfit, grad = eng.misfit_and_gradient(obs.to(eng.device), mask=mask,
                                               guard_radius=guard_radius)
    except FloatingPointError as exc:
        raise NumericError(str(exc)) from exc
    g = grad.cpu().numpy()
    return [float(m) for m in misfit.cpu().numpy()], [GradientMap(grid, g[b]) for b in range(B)]


def fd_gradient_oracle(sos: SosMap, m_obs: ChannelData, pulse: SourcePulse, cells, eps: float,
                       damping: DampingProfile | None = None, *, density=None) -> np.ndarray:
    """Central-difference misfit derivatives at selected cells (adjoint.py:154-186).

    All 2*len(cells) perturbed models run as phantoms of ONE batched forward
    sweep on the device with arith="f64" (the sweep itself in f64: a misfit
    difference needs more than the f32 kernels' 5e-7 trace error); each misfit
    sum((obs - sim)^2) is reduced in f64 by the residual kernel.  Noise floor: the receiver samples leave the sweep as
    f32 (the ChannelData format of the engine), so each misfit carries a
    relative rounding error of order 1e-7 * (trace/residual energy ratio);
    choose ``eps`` so that the misfit change 2*eps*|g| stays well above it
    (the reference's own grad-check case, eps = 1e-3 m/s on its 16x16 grid,
    is checked against the reference's values in tests/test_gpu_api_extras.py).
    """
    import torch

    if eps <= 0:
        raise ValueError("eps must be positive")
    geometry = m_obs.geometry
    damping = damping if damping is not None else zero_damping(sos.grid)
    cells = [tuple(int(v) for v in c) for c in cells]
    if not cells:
        return np.empty(0)
    base = np.array(sos.values)
    maps = []
    for ix, iz in cells:
        plus = np.array(base)
        plus[ix, iz] += eps
        minus = np.array(base)
        minus[ix, iz] -= eps
        for m in (plus, minus):
            _check_simulation_inputs(sos.with_values(m), geometry, pulse, damping)
            maps.append(m)
    rho = _density_values(density, sos.grid)
    B = len(maps)
    eng = get_engine(sos.grid, geometry.tx_nodes(), geometry.rx_nodes(), geometry.element_nodes,
                     pulse.samples, damping, n_phantoms=B, has_rho=rho is not None, arith="f64")
    eng.set_model(np.stack(maps), None if rho is None else np.broadcast_to(rho, (B,) + rho.shape))
    obs = torch.as_tensor(np.ascontiguousarray(m_obs.traces), dtype=torch.float64).to(eng.device)
    obs = obs.repeat(B, 1, 1)
    try:
        j = eng.misfit(obs).cpu().numpy()
    except FloatingPointError as exc:
        raise NumericError(str(exc)) from exc
    return (j[0::2] - j[1::2]) / (2.0 * eps)
