"""Classical ADMM-TV waveform inversion on the GPU physics step.

Mirror of the reference's baseline solver (fwi.py:1-271): scaled-dual ADMM on
min_C misfit(C) + lambda TV(Z) s.t. C = Z, with a fixed-step L-BFGS inner solve
of the augmented data term, an anisotropic-TV proximal step (dual projected
gradient) and dual ascent — same names, defaults, operation order and error
types.  Every iterate stays on the device: the data term is the libdufwi
forward + adjoint (one C-ABI launch set per evaluation), and the L-BFGS two-loop
recursion, TV prox and ADMM updates are float64 tensor operations (the
elementwise ones in the reference's order, so ``tv_prox`` gives the
reference's bits on identical input).

``admm_fwi_batch`` inverts B phantoms that share one acquisition at once:
every data-term evaluation is one launch set over B x S units, and the
L-BFGS state is kept per phantom (curvature pairs accepted, evicted and used
per phantom exactly as in the single-phantom recursion).  ``admm_fwi`` is its
B = 1 case with the reference signature.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Callable

import numpy as np
import torch

from .forward import (DampingProfile, NumericError, SourcePulse, _check_simulation_inputs,
                      get_engine, zero_damping)
from .grid import ChannelData, SosMap, check_cfl

__all__ = ["FwiConfig", "FwiDivergenceError", "tv_prox", "total_variation", "lbfgs_minimize",
           "lbfgs_minimize_batch", "admm_fwi", "admm_fwi_batch", "plain_gradient_descent"]


class FwiDivergenceError(RuntimeError):
    """Inner solve produced a non-finite misfit (fwi.py:31-36)."""

    def __init__(self, outer_iteration: int):
        super().__init__(f"inner solve diverged at outer iteration {outer_iteration}")
        self.outer_iteration = outer_iteration


@dataclass(frozen=True)
class FwiConfig:
    """ADMM-FWI settings (fwi.py:39-67); ``rho_admm=None`` picks
    1e-2 misfit(C0)/||C0||^2 at run time, ``tv_weight=None`` defaults to rho."""

    outer_iters: int = 200
    inner_lbfgs_iters: int = 5
    inner_lr: float = 1.0
    tv_weight: float | None = None
    rho_admm: float | None = None
    bounds: tuple[float, float] = (1300.0, 3200.0)

    def __post_init__(self):
        if self.outer_iters < 1:
            raise ValueError("outer_iters must be >= 1")
        if self.inner_lbfgs_iters < 1:
            raise ValueError("inner_lbfgs_iters must be >= 1")
        if self.tv_weight is not None and self.tv_weight < 0:
            raise ValueError("tv_weight must be >= 0")
        if self.rho_admm is not None and self.rho_admm <= 0:
            raise ValueError("rho_admm must be > 0")
        if not self.bounds[0] < self.bounds[1]:
            raise ValueError("bounds must satisfy c_min < c_max")


# ------------------------------------------------------------------- TV prox
def _div(zx: torch.Tensor, zz: torch.Tensor, shape) -> torch.Tensor:
    """Negative adjoint of the forward difference (fwi.py:78-85), trailing two axes."""
    out = torch.zeros(shape, dtype=zx.dtype, device=zx.device)
    out[..., :-1, :] -= zx
    out[..., 1:, :] += zx
    out[..., :, :-1] -= zz
    out[..., :, 1:] += zz
    return out


def _tv_prox_t(v: torch.Tensor, weight: torch.Tensor, iters: int) -> torch.Tensor:
    """Batched prox of weight_b * TV at v_b (fwi.py:94-117); weight (B,) >= 0."""
    w = weight.reshape(-1, 1, 1).to(v.dtype)
    zero = w == 0
    ws = torch.where(zero, torch.ones_like(w), w)  # keep the arithmetic finite; masked below
    zx = torch.zeros(v.shape[:-2] + (v.shape[-2] - 1, v.shape[-1]), dtype=v.dtype, device=v.device)
    zz = torch.zeros(v.shape[:-2] + (v.shape[-2], v.shape[-1] - 1), dtype=v.dtype, device=v.device)
    # divisor materialised full size: a broadcast scalar divisor may be turned into a
    # multiplication by its reciprocal, which is not the reference's IEEE division
    d8 = (8.0 * ws).expand(v.shape).contiguous()
    for _ in range(iters):
        x = v - ws * _div(zx, zz, v.shape)
        zx = torch.clamp(zx + (x[..., 1:, :] - x[..., :-1, :]) / d8[..., 1:, :], -1.0, 1.0)
        zz = torch.clamp(zz + (x[..., :, 1:] - x[..., :, :-1]) / d8[..., :, 1:], -1.0, 1.0)
    out = v - ws * _div(zx, zz, v.shape)
    return torch.where(zero, v, out)


def tv_prox(v, weight: float, iters: int = 20):
    """Approximate prox of ``weight * TV`` at ``v`` (fwi.py:94-117); numpy or tensor."""
    if weight < 0:
        raise ValueError("weight must be >= 0")
    is_np = not isinstance(v, torch.Tensor)
    t = torch.as_tensor(np.asarray(v, dtype=np.float64)) if is_np else v.to(torch.float64)
    if weight == 0.0:
        out = t.clone()
    else:
        out = _tv_prox_t(t[None], torch.tensor([float(weight)], dtype=torch.float64, device=t.device),
                         iters)[0]
    return out.cpu().numpy() if is_np else out


def total_variation(v) -> float:
    """Anisotropic TV: l1 norm of both forward differences (fwi.py:88-91)."""
    t = torch.as_tensor(np.asarray(v, dtype=np.float64)) if not isinstance(v, torch.Tensor) else v
    return float((t[1:, :] - t[:-1, :]).abs().sum() + (t[:, 1:] - t[:, :-1]).abs().sum())


# -------------------------------------------------------------------- L-BFGS
def _dot(a: torch.Tensor, b: torch.Tensor) -> torch.Tensor:
    return (a * b).flatten(1).sum(dim=1)


def _bc(s: torch.Tensor, like: torch.Tensor) -> torch.Tensor:
    return s.reshape((-1,) + (1,) * (like.dim() - 1))


def lbfgs_minimize_batch(value_grad_fn, x0: torch.Tensor, iters: int, lr: float, memory: int = 5,
                         project=None):
    """Batched fixed-step L-BFGS (fwi.py:120-183), one independent recursion per
    leading index.  ``value_grad_fn(x)`` returns (f (B,), g like x).  Pairs with
    s.y <= 1e-12 are skipped and the oldest evicted beyond ``memory``, per phantom.
    Returns (x, values list of (B,) tensors)."""
    x = x0.clone()
    S, Y, V = [], [], []  # stored pairs and their per-phantom validity (B,) bool
    f, g = value_grad_fn(x)
    values = [f]
    for it in range(iters):
        bad = ~torch.isfinite(f) | ~torch.isfinite(g).flatten(1).all(dim=1)
        if bool(bad.any()):
            err = FloatingPointError(f"non-finite objective at inner step {it}")
            err.phantoms = torch.nonzero(bad).flatten().tolist()
            raise err
        have = torch.zeros_like(f, dtype=torch.bool)
        for v in V:
            have |= v
        # two-loop recursion over the valid pairs of each phantom, newest first
        q = g.clone()
        alphas, rhos = [], []
        for s, y, v in zip(reversed(S), reversed(Y), reversed(V)):
            rho = torch.where(v, 1.0 / torch.where(v, _dot(y, s), torch.ones_like(f)),
                              torch.zeros_like(f))
            alpha = rho * _dot(s, q)
            q = q - _bc(alpha, q) * y
            alphas.append(alpha)
            rhos.append(rho)
        # gamma from each phantom's most recent valid pair
        gamma = torch.ones_like(f)
        found = torch.zeros_like(have)
        for s, y, v in zip(reversed(S), reversed(Y), reversed(V)):
            take = v & ~found
            gamma = torch.where(take, _dot(s, y) / torch.where(take, _dot(y, y), torch.ones_like(f)),
                                gamma)
            found |= v
        r = _bc(gamma, q) * q
        for (s, y), alpha, rho in zip(zip(S, Y), reversed(alphas), reversed(rhos)):
            beta = rho * _dot(y, r)
            r = r + _bc(alpha - beta, r) * s
        g1 = g.abs().flatten(1).sum(dim=1)
        scale = torch.where(g1 > 0, torch.clamp(1.0 / torch.where(g1 > 0, g1, torch.ones_like(g1)),
                                                max=1.0), torch.ones_like(g1))
        direction = torch.where(_bc(have, g), -r, -g * _bc(scale, g))
        x_new = x + lr * direction
        if project is not None:
            x_new = project(x_new)
        f_new, g_new = value_grad_fn(x_new)
        s = x_new - x
        y = g_new - g
        acc = _dot(y, s) > 1e-12
        if bool(acc.any()):
            S.append(s)
            Y.append(y)
            V.append(acc.clone())
            # per-phantom eviction of the oldest valid pair beyond ``memory``
            count = torch.stack(V).sum(dim=0)
            over = count > memory
            if bool(over.any()):
                for v in V:
                    first = v & over
                    v &= ~first
                    over &= ~first
            while V and not bool(V[0].any()):
                S.pop(0), Y.pop(0), V.pop(0)
        x, f, g = x_new, f_new, g_new
        values.append(f)
    return x, values


def lbfgs_minimize(value_grad_fn: Callable, x0, iters: int, lr: float, memory: int = 5,
                   project: Callable | None = None):
    """Reference signature (fwi.py:120-127): numpy in, numpy out, one problem."""
    def fn(xb):
        f, g = value_grad_fn(xb[0].cpu().numpy())
        return (torch.tensor([float(f)], dtype=torch.float64),
                torch.as_tensor(np.asarray(g, dtype=np.float64))[None])

    proj = None
    if project is not None:
        proj = lambda xb: torch.as_tensor(np.asarray(project(xb[0].numpy()), np.float64))[None]  # noqa: E731
    x, vals = lbfgs_minimize_batch(fn, torch.as_tensor(np.array(x0, dtype=np.float64))[None],
                                   iters, lr, memory, proj)
    return x[0].numpy(), [float(v[0]) for v in vals]


# -------------------------------------------------------------------- drivers
class _DataTerm:
    """misfit_and_gradient of B phantoms on one acquisition, device tensors in and out."""

    def __init__(self, m_obs_list, grid, pulse: SourcePulse, damping: DampingProfile):
        geom = m_obs_list[0].geometry
        for m in m_obs_list:
            if not m.geometry.same_acquisition(geom):
                raise ValueError("batched FWI needs one acquisition geometry")
        self.grid = grid
        self.eng = get_engine(grid, geom.tx_nodes(), geom.rx_nodes(), geom.element_nodes,
                              pulse.samples, damping, n_phantoms=len(m_obs_list), arith="f64")
        self.obs = torch.from_numpy(np.concatenate(
            [np.require(m.traces, np.float64, ["C", "W"]) for m in m_obs_list])).to(self.eng.device)
        self.limit = grid.dx / (grid.dt * np.sqrt(2.0))  # check_cfl bound (grid.py:242-251)

    def __call__(self, c: torch.Tensor):
        cmax = float(c.max())
        if not check_cfl(self.grid, cmax).ok:
            raise ValueError(f"CFL violated by an iterate: c_max={cmax} m/s")
        self.eng.set_model(c)
        mis, g = self.eng.misfit_and_gradient(self.obs, check_finite=False)
        return mis, g


def admm_fwi_batch(m_obs_list, c0_list, cfg: FwiConfig, pulse: SourcePulse,
                   damping: DampingProfile | None = None, callback=None):
    """ADMM-TV inversion of B phantoms at once (fwi.py:191-248 per phantom).
    Returns (list of final SosMaps, list of per-phantom misfit logs)."""
    grid = c0_list[0].grid
    damping = damping if damping is not None else zero_damping(grid)
    for m, c in zip(m_obs_list, c0_list):
        _check_simulation_inputs(c, m.geometry, pulse, damping)
    data = _DataTerm(m_obs_list, grid, pulse, damping)
    dev = data.eng.device
    c = torch.as_tensor(np.stack([np.asarray(c.values, np.float64) for c in c0_list]), device=dev)
    c_min, c_max = cfg.bounds

    misfit0, _ = data(c)
    if not bool(torch.isfinite(misfit0).all()):
        raise NumericError("non-finite misfit at the starting model")
    rho = (torch.full_like(misfit0, cfg.rho_admm) if cfg.rho_admm is not None
           else 1e-2 * misfit0 / (c * c).flatten(1).sum(dim=1))
    lam = torch.full_like(rho, cfg.tv_weight) if cfg.tv_weight is not None else rho
    z = c.clone()
    w = torch.zeros_like(c)
    logs = [misfit0.clone()]
    for outer in range(cfg.outer_iters):
        def augmented(values):
            mis, grad = data(values)
            diff = values - z + w
            return mis + 0.5 * rho * (diff * diff).flatten(1).sum(dim=1), grad + _bc(rho, diff) * diff

        try:
            c, _ = lbfgs_minimize_batch(augmented, c, cfg.inner_lbfgs_iters, cfg.inner_lr,
                                        project=lambda x: torch.clamp(x, c_min, c_max))
        except FloatingPointError as exc:
            raise FwiDivergenceError(outer) from exc
        c = torch.clamp(c, c_min, c_max)
        z = _tv_prox_t(c + w, lam / rho, 20)
        w = w + c - z
        mis, _ = data(c)
        if not bool(torch.isfinite(mis).all()):
            raise FwiDivergenceError(outer)
        logs.append(mis.clone())
        if callback is not None:
            callback(outer, mis.cpu().numpy())
    host = c.cpu().numpy()
    log = torch.stack(logs).cpu().numpy()
    return ([c0.with_values(host[b]) for b, c0 in enumerate(c0_list)],
            [log[:, b].tolist() for b in range(len(c0_list))])


def admm_fwi(m_obs: ChannelData, c0: SosMap, cfg: FwiConfig, pulse: SourcePulse,
             damping: DampingProfile | None = None, callback=None):
    """Run the ADMM-TV inversion for exactly ``cfg.outer_iters`` iterations
    (fwi.py:191-248); returns (final map, [misfit0, misfit after each outer])."""
    cb = None if callback is None else (lambda k, mis: callback(k, float(mis[0])))
    maps, logs = admm_fwi_batch([m_obs], [c0], cfg, pulse, damping, cb)
    return maps[0], logs[0]


def plain_gradient_descent(m_obs: ChannelData, c0: SosMap, steps: int, gamma: float,
                           pulse: SourcePulse, damping: DampingProfile | None = None,
                           bounds: tuple[float, float] | None = None) -> SosMap:
    """Fixed-step descent C <- C - gamma g on the data misfit (fwi.py:251-271)."""
    grid = c0.grid
    damping = damping if damping is not None else zero_damping(grid)
    _check_simulation_inputs(c0, m_obs.geometry, pulse, damping)
    data = _DataTerm([m_obs], grid, pulse, damping)
    c = torch.as_tensor(np.asarray(c0.values, np.float64), device=data.eng.device)[None]
    for _ in range(steps):
        _, g = data(c)
        if not bool(torch.isfinite(g).all()):
            raise FloatingPointError("non-finite gradient")
        c = c - gamma * g
        if bounds is not None:
            c = torch.clamp(c, bounds[0], bounds[1])
    return c0.with_values(c[0].cpu().numpy())
