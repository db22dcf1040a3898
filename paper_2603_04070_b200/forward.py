"""Forward modelling API (mirror of ``fwilab.forward``) on the sm_100a kernels.

Scheme (forward.py:1-15 of the reference):

    U[t] = (2 - D^2 dt^2)/(1 + D dt) U[t-1] + (D dt - 1)/(1 + D dt) U[t-2]
         + c^2 dt^2/(1 + D dt) lap(U[t-1]) + S[t]

with the 5-point Laplacian, zero outside the grid, and the polynomial damping
band ``D``.  Public entry points keep the reference signatures; the extra
keyword ``density=`` selects the variable-density operator
``rho div(1/rho grad u)``.  Every sweep runs in ``libdufwi.so`` — there is no
CPU path here.
"""

from __future__ import annotations

import hashlib
import math
import warnings
from collections import OrderedDict
from dataclasses import dataclass

import numpy as np

from .grid import (AcquisitionGeometry, ChannelData, DensityMap, GeometryError, Grid2D, SosMap,
                   check_cfl)

__all__ = ["PML_REFERENCE_SPEED", "NumericError", "DampingProfile", "zero_damping", "build_pml",
           "SourcePulse", "make_source_pulse", "Wavefield", "laplacian", "step_wavefield",
           "simulate_wavefield", "simulate_transmission", "simulate_all", "get_engine"]

#: damping calibration speed (forward.py:47-48)
PML_REFERENCE_SPEED = 1500.0


class NumericError(ValueError):
    """Non-finite values in a solver input or state (forward.py:51-52)."""


@dataclass(frozen=True)
class DampingProfile:
    """Damping coefficients in 1/s (forward.py:55-74).

    ``profiles`` (extension) keeps the separable axis ramps of :func:`build_pml`
    so the kernels read two 1-D arrays instead of the 2-D map; the values are
    identical (``max(px[i], pz[j])``).
    """

    grid: Grid2D
    values: np.ndarray
    profiles: tuple[np.ndarray, np.ndarray] | None = None

    def __post_init__(self):
        v = np.asarray(self.values, dtype=np.float64)
        if v.shape != self.grid.shape:
            raise ValueError(f"damping shape {v.shape} != grid {self.grid.shape}")
        if not np.isfinite(v).all() or v.min() < 0.0:
            raise ValueError("damping must be finite and non-negative")
        v = np.ascontiguousarray(v)
        v.flags.writeable = False
        object.__setattr__(self, "values", v)
        if self.profiles is None:
            object.__setattr__(self, "profiles", _separable_profiles(v))

    def interior_mask(self) -> np.ndarray:
        return self.values == 0.0


def _separable_profiles(v: np.ndarray):
    """Axis ramps (px, pz) with max(px[i], pz[j]) == v exactly, or None.

    A map built like build_pml's (forward.py:135-137) but handed over as plain
    values (e.g. loaded from disk) is recognised, so the kernels read the two
    1-D ramps: with an undamped cell (i0, j0), px = v[:, j0] and pz = v[i0, :]."""
    zeros = np.argwhere(v == 0.0)
    if zeros.size == 0:
        return None
    i0, j0 = zeros[0]
    px, pz = v[:, j0].copy(), v[i0, :].copy()
    if not np.array_equal(np.maximum(px[:, None], pz[None, :]), v):
        return None
    return px, pz


def zero_damping(grid: Grid2D) -> DampingProfile:
    return DampingProfile(grid, np.zeros(grid.shape), (np.zeros(grid.nx), np.zeros(grid.nz)))


def build_pml(grid: Grid2D, thickness: int, target_attenuation: float = 1e-3,
              exponent: float = 2.0) -> DampingProfile:
    """Polynomial absorbing band, corners = max of the axis ramps (forward.py:81-137).

    ``D_max = -ln(a) c_ref (m+1) / (2 T dx)``; ``D(d) = D_max ((T-d)/T)^m``.
    """
    if thickness < 0:
        raise ValueError("thickness must be non-negative")
    if thickness == 0:
        return zero_damping(grid)
    if 2 * thickness >= min(grid.nx, grid.nz):
        raise GeometryError(
            f"PML of {thickness} cells does not leave an interior on a {grid.nx}x{grid.nz} grid")
    if not 0.0 < target_attenuation < 1.0:
        raise ValueError("target_attenuation must lie in (0, 1)")
    d_max = (-math.log(target_attenuation) * PML_REFERENCE_SPEED * (exponent + 1.0)
             / (2.0 * thickness * grid.dx))
    if d_max * grid.dt >= 2.0:
        warnings.warn(f"peak damping D*dt = {d_max * grid.dt:.2f} >= 2 destabilizes the explicit "
                      "scheme; use a thicker band or a smaller time step", stacklevel=2)

    def ramp(n: int) -> np.ndarray:
        k = np.arange(n)
        d = np.minimum(k, n - 1 - k).astype(np.float64)
        return d_max * np.clip((thickness - d) / thickness, 0.0, None) ** exponent

    px, pz = ramp(grid.nx), ramp(grid.nz)
    return DampingProfile(grid, np.maximum(px[:, None], pz[None, :]), (px, pz))


@dataclass(frozen=True)
class SourcePulse:
    """Discrete source waveform (forward.py:140-160)."""

    samples: np.ndarray
    dt: float
    f_c: float

    def __post_init__(self):
        s = np.asarray(self.samples, dtype=np.float64)
        if s.ndim != 1:
            raise ValueError("pulse samples must be 1-D")
        if not np.isfinite(s).all():
            raise ValueError("pulse contains non-finite samples")
        s = np.ascontiguousarray(s)
        s.flags.writeable = False
        object.__setattr__(self, "samples", s)

    @property
    def nt(self) -> int:
        return int(self.samples.shape[0])


def make_source_pulse(f_c: float, dt: float, nt: int, kind: str = "gaussian_derivative") -> SourcePulse:
    """Gaussian / derivative-of-Gaussian, sigma = 1/(2 pi f_c), t0 = 7 sigma (forward.py:163-199)."""
    if f_c <= 0 or dt <= 0 or nt < 1:
        raise ValueError("f_c, dt must be positive and nt >= 1")
    if f_c * dt >= 0.5:
        raise ValueError(f"center frequency {f_c} Hz violates Nyquist at dt={dt} s")
    sigma = 1.0 / (2.0 * math.pi * f_c)
    t0 = 7.0 * sigma
    t = np.arange(nt) * dt
    if nt * dt < t0 + 5.0 * sigma:
        warnings.warn("time window is shorter than the pulse support; the waveform will be "
                      "truncated", stacklevel=2)
    env = np.exp(-((t - t0) ** 2) / (2.0 * sigma ** 2))
    if kind == "gaussian":
        w = env
    elif kind == "gaussian_derivative":
        w = -(t - t0) / sigma ** 2 * env
    else:
        raise ValueError(f"unknown pulse kind {kind!r}")
    peak = np.abs(w).max()
    return SourcePulse(w / peak if peak > 0 else w, dt, f_c)


@dataclass
class Wavefield:
    """Rolling two-step history (forward.py:202-208)."""

    u_curr: np.ndarray
    u_prev: np.ndarray
    t: int


# ------------------------------------------------------------ field utilities
def _device():
    import torch

    from . import _lib

    _lib.lib()  # fails loudly without the extension
    if not torch.cuda.is_available():
        raise _lib.ExtensionUnavailable("no CUDA device visible; the DUFWI path is GPU-only")
    return torch.device("cuda", torch.cuda.current_device())


def laplacian(u: np.ndarray, dx: float) -> np.ndarray:
    """5-point Laplacian with zeros outside the grid on the trailing two axes
    (forward.py:211-223), computed by ``dufwi_laplacian`` in float64 with the
    reference's accumulation order (bit-identical).  Returns float64."""
    import torch

    from . import _lib

    a = np.asarray(u, dtype=np.float64)
    if a.ndim < 2:
        raise ValueError("laplacian needs at least two axes")
    nx, nz = a.shape[-2:]
    batch = int(np.prod(a.shape[:-2], dtype=np.int64))
    if a.size == 0:
        return np.zeros(a.shape)
    dev = _device()
    src = torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    out = torch.empty_like(src)
    _lib.check(_lib.lib().dufwi_laplacian(src.data_ptr(), batch, nx, nz, float(dx), out.data_ptr(),
                                          torch.cuda.current_stream(dev).cuda_stream))
    return out.cpu().numpy()


def step_wavefield(u_prev: np.ndarray, u_prev2: np.ndarray, sos: SosMap,
                   damping: DampingProfile, s_t, dt: float) -> np.ndarray:
    """Single explicit time step (forward.py:237-253), same checks and exceptions;
    the update runs in ``dufwi_step_field`` (f64, bit-identical to NumPy)."""
    import torch

    from . import _lib

    if np.shape(u_prev) != sos.grid.shape or np.shape(u_prev2) != sos.grid.shape:
        raise ValueError("wavefield shape does not match the grid")
    for name, arr in (("u_prev", u_prev), ("u_prev2", u_prev2), ("s_t", s_t)):
        if not np.all(np.isfinite(arr)):
            raise NumericError(f"non-finite values in {name}")
    grid = sos.grid
    dev = _device()

    def up(a):
        return torch.from_numpy(np.ascontiguousarray(
            np.broadcast_to(np.asarray(a, dtype=np.float64), grid.shape))).to(dev)

    u1, u2, c, d, s = (up(a) for a in (u_prev, u_prev2, sos.values, damping.values, s_t))
    out = torch.empty_like(u1)
    _lib.check(_lib.lib().dufwi_step_field(u1.data_ptr(), u2.data_ptr(), c.data_ptr(), d.data_ptr(),
                                           s.data_ptr(), grid.nx, grid.nz, float(grid.dx),
                                           float(dt), out.data_ptr(),
                                           torch.cuda.current_stream(dev).cuda_stream))
    return out.cpu().numpy()


# ---------------------------------------------------------------- engine cache
_ENGINE_CACHE: "OrderedDict[str, object]" = OrderedDict()
_ENGINE_CACHE_SIZE = 4


_ARRAY_DIGESTS: OrderedDict = OrderedDict()  # id -> (array, digest) of large read-only arrays


def _array_digest(p: np.ndarray) -> bytes:
    """sha1 of an array's dtype, shape and bytes; memoised for large read-only
    arrays (the immutable containers' damping maps and pulses), which keeps the
    engine lookup of a repeated public-API call off the host's critical path.
    The memo holds a reference, so an id is never reused while it is cached."""
    memo = p.nbytes >= 4096 and not p.flags.writeable
    if memo:
        hit = _ARRAY_DIGESTS.get(id(p))
        if hit is not None and hit[0] is p:
            return hit[1]
    h = hashlib.sha1(str((p.dtype, p.shape)).encode())
    h.update(np.ascontiguousarray(p).tobytes())
    d = h.digest()
    if memo:
        _ARRAY_DIGESTS[id(p)] = (p, d)
        while len(_ARRAY_DIGESTS) > 32:
            _ARRAY_DIGESTS.popitem(last=False)
    return d


def _digest(*parts) -> str:
    h = hashlib.sha1()
    for p in parts:
        if isinstance(p, np.ndarray):
            h.update(_array_digest(p))
        else:
            h.update(repr(p).encode())
    return h.hexdigest()


def get_engine(grid: Grid2D, tx_nodes, rx_nodes, element_nodes, pulse: np.ndarray,
               damping: DampingProfile, n_phantoms: int = 1, has_rho: bool = False,
               engine: str = "auto", arith: str = "f32"):
    """Cached :class:`~paper_2603_04070_b200.engine.PhysicsEngine` for an acquisition.

    ``arith``: "f32" (default; the increment-form f32 kernels, inside the north-star
    tolerances) or "f64" (the reference's operation order in f64; misfit differencing
    and convergence studies, include/dufwi.h DUFWI_ARITH_*)."""
    import torch

    from .engine import PhysicsEngine

    dev = torch.cuda.current_device() if torch.cuda.is_available() else -1
    key = _digest(grid, np.asarray(tx_nodes), np.asarray(rx_nodes), np.asarray(element_nodes),
                  np.asarray(pulse), damping.values, n_phantoms, has_rho, engine, arith, dev)
    eng = _ENGINE_CACHE.get(key)
    if eng is None:
        prof = damping.profiles
        eng = PhysicsEngine(nx=grid.nx, nz=grid.nz, nt=grid.nt, dx=grid.dx, dt=grid.dt,
                            tx_nodes=tx_nodes, rx_nodes=rx_nodes, element_nodes=element_nodes,
                            pulse=pulse, damping_profiles=prof,
                            damping_values=None if prof is not None else damping.values,
                            n_phantoms=n_phantoms, has_rho=has_rho, engine=engine, arith=arith)
        _ENGINE_CACHE[key] = eng
        while len(_ENGINE_CACHE) > _ENGINE_CACHE_SIZE:
            _ENGINE_CACHE.popitem(last=False)
    else:
        _ENGINE_CACHE.move_to_end(key)
    return eng


def _check_simulation_inputs(sos: SosMap, geometry: AcquisitionGeometry, pulse: SourcePulse,
                             damping: DampingProfile) -> None:
    """Same checks and exception types as forward.py:256-270."""
    if geometry.grid != sos.grid:
        raise ValueError("geometry and speed map use different grids")
    cfl = check_cfl(sos.grid, sos.c_max)
    if not cfl.ok:
        raise ValueError(f"CFL violated: ratio {cfl.ratio:.4f} > 1 for c_max={sos.c_max} m/s")
    if pulse.nt != sos.grid.nt:
        raise ValueError("pulse length does not match grid.nt")
    nodes = geometry.element_nodes
    if np.any(damping.values[nodes[:, 0], nodes[:, 1]] > 0.0):
        raise GeometryError("transducer elements lie inside the damping band")


def _density_values(density, grid):
    if density is None:
        return None
    d = density.values if isinstance(density, DensityMap) else np.asarray(density, dtype=np.float64)
    if d.shape != grid.shape:
        raise ValueError("density shape does not match the grid")
    return d


def _run_forward(sos, geometry, pulse, damping, density, tx, rx, arith="f32"):
    eng = get_engine(sos.grid, tx, rx, geometry.element_nodes, pulse.samples, damping,
                     has_rho=density is not None, arith=arith)
    eng.set_model(sos.values[None], None if density is None else density[None])
    try:
        return eng.forward()
    except FloatingPointError as exc:
        raise NumericError(str(exc)) from exc


def simulate_all(sos: SosMap, geometry: AcquisitionGeometry, pulse: SourcePulse,
                 damping: DampingProfile | None = None, *, density=None,
                 arith: str = "f32") -> ChannelData:
    """Channel data for every transmission in transmission order (forward.py:355-369).

    ``arith="f64"`` runs the sweep in float64 in the reference's operation order
    (default: the f32 increment form, traces within ~5e-7 of it)."""
    damping = damping if damping is not None else zero_damping(sos.grid)
    _check_simulation_inputs(sos, geometry, pulse, damping)
    rho = _density_values(density, sos.grid)
    tr = _run_forward(sos, geometry, pulse, damping, rho, geometry.tx_nodes(), geometry.rx_nodes(),
                      arith)
    return ChannelData(tr.double().cpu().numpy(), geometry, sos.grid.dt)


def simulate_transmission(sos: SosMap, geometry: AcquisitionGeometry, pulse: SourcePulse, p: int,
                          damping: DampingProfile | None = None, *, density=None,
                          arith: str = "f32") -> np.ndarray:
    """Traces (nt, n_r) of transmission ``p`` (forward.py:335-352)."""
    if not 0 <= p < geometry.n_p:
        raise ValueError(f"transmission index {p} out of range [0, {geometry.n_p})")
    damping = damping if damping is not None else zero_damping(sos.grid)
    _check_simulation_inputs(sos, geometry, pulse, damping)
    rho = _density_values(density, sos.grid)
    tx = geometry.tx_nodes()[p:p + 1]
    rx = geometry.rx_nodes()[p:p + 1]
    tr = _run_forward(sos, geometry, pulse, damping, rho, tx, rx, arith)
    return tr[0].T.double().cpu().numpy().copy()


def simulate_wavefield(sos: SosMap, pulse: SourcePulse, source_node: tuple[int, int],
                       damping: DampingProfile | None = None, *, density=None) -> np.ndarray:
    """Full field history (nt, nx, nz) of one point source (forward.py:316-332)."""
    damping = damping if damping is not None else zero_damping(sos.grid)
    cfl = check_cfl(sos.grid, sos.c_max)
    if not cfl.ok:
        raise ValueError(f"CFL violated: ratio {cfl.ratio:.4f} > 1")
    rho = _density_values(density, sos.grid)
    tx = np.asarray([source_node], dtype=np.int64)
    eng = get_engine(sos.grid, tx, tx[:, None, :], tx, pulse.samples, damping,
                     has_rho=rho is not None)
    eng.set_model(sos.values[None], None if rho is None else rho[None])
    hist = eng.wavefield_history(0)
    out = hist.double().cpu().numpy()
    if not np.isfinite(out[-1]).all():
        raise NumericError("simulation diverged: non-finite wavefield")
    return out
