"""Seeded synthetic workloads for BASELINE.json configs 0-4.

No public dataset is used: every phantom, array and pulse here is generated
from ``numpy.random.default_rng(seed)`` with the shapes, sizes and value
distributions the configs state.  Conventions:

* G2 — the stated grid size is the *interior*; the PML is padded outside, so
  the simulated grid is ``n + 2*pml`` per side and cell updates are counted on
  that padded grid.
* G1 — the linear array sits on the first interior row ``z = pml`` with pitch
  2 cells, centred along x; transmits are a subset of its elements.
* G4 — the pulse is a Gaussian-modulated sinusoid
  ``sin(2 pi f (t-t0)) exp(-((t-t0) f)^2)``, ``t0 = 2/f``, peak-normalised.
* G6 — unstated values assumed: config 2 dt 20 ns / 1 MHz, config 4 dt 10 ns /
  2.5 MHz; speckle ``c *= 1 + 0.01 N(0,1)`` per cell.
* G7 — DUFWI starts from the homogeneous 1540 m/s map.
"""

from __future__ import annotations

from dataclasses import dataclass, field, asdict

import numpy as np

__all__ = ["WorkloadSpec", "CONFIGS", "get_config", "gaussian_sine_pulse",
           "linear_array", "inclusion_phantom", "make_workload", "Workload"]


@dataclass(frozen=True)
class WorkloadSpec:
    name: str
    n_interior: int
    pml: int
    dx: float
    dt: float
    nt: int
    f_c: float
    n_elements: int
    n_tx: int
    tx_stride: int | None          # None: evenly spaced round(linspace)
    n_rx: int
    n_phantoms: int
    k_stages: int
    inclusions: tuple[int, int]    # min/max count
    shape: str                     # "disk" | "ellipse"
    radius_cells: tuple[float, float]
    contrast: float                # +/- m/s
    density: bool
    speckle: float
    background: float = 1540.0
    rho0: float = 1000.0
    rho_range: tuple[float, float] = (950.0, 1100.0)
    strips: bool = False           # boundary-strip reconstruction (config 3/4)

    @property
    def n(self) -> int:
        return self.n_interior + 2 * self.pml

    def units(self) -> int:
        return self.n_tx * self.n_phantoms

    def as_dict(self) -> dict:
        return asdict(self)


CONFIGS: dict[int, WorkloadSpec] = {
    0: WorkloadSpec("config0-gradient", 128, 16, 1e-4, 2e-8, 1000, 1e6, 64, 8, None, 64,
                    1, 0, (3, 3), "disk", (8.0, 20.0), 40.0, False, 0.0),
    1: WorkloadSpec("config1-dufwi-k5", 128, 16, 1e-4, 2e-8, 1000, 1e6, 64, 8, None, 64,
                    1, 5, (3, 3), "disk", (8.0, 20.0), 40.0, False, 0.0),
    2: WorkloadSpec("config2-dufwi-rho", 256, 20, 1e-4, 2e-8, 2000, 1e6, 128, 32, None, 128,
                    8, 5, (1, 6), "ellipse", (10.0, 40.0), 60.0, True, 0.01),
    3: WorkloadSpec("config3-strips", 512, 24, 5e-5, 1e-8, 4000, 2.5e6, 256, 128, 2, 256,
                    1, 3, (1, 6), "ellipse", (10.0, 40.0), 60.0, True, 0.01, strips=True),
    # config 4 names "random multi-inclusion SoS phantoms": speed of sound only
    4: WorkloadSpec("config4-scaling", 1024, 32, 5e-5, 1e-8, 6000, 2.5e6, 256, 256, 1, 256,
                    4, 0, (1, 6), "ellipse", (10.0, 40.0), 60.0, False, 0.01, strips=True),
}


def get_config(i: int) -> WorkloadSpec:
    return CONFIGS[int(i)]


def gaussian_sine_pulse(f_c: float, dt: float, nt: int) -> np.ndarray:
    """Peak-normalised Gaussian-modulated sinusoid, two cycles of support each side."""
    t = np.arange(nt) * dt
    t0 = 2.0 / f_c
    s = np.sin(2.0 * np.pi * f_c * (t - t0)) * np.exp(-(((t - t0) * f_c) ** 2))
    return s / np.abs(s).max()


def linear_array(spec: WorkloadSpec):
    """Element nodes (E,2), transmit element indices (S,), receive pattern (S,R)."""
    span = 2 * (spec.n_elements - 1) + 1
    x0 = spec.pml + (spec.n_interior - span) // 2
    ex = x0 + 2 * np.arange(spec.n_elements)
    nodes = np.stack([ex, np.full_like(ex, spec.pml)], axis=1).astype(np.int64)
    if spec.tx_stride is None:
        tx = np.rint(np.linspace(0, spec.n_elements - 1, spec.n_tx)).astype(np.int64)
    else:
        tx = (np.arange(spec.n_tx) * spec.tx_stride).astype(np.int64)
    if spec.n_rx == spec.n_elements:
        rx = np.tile(np.arange(spec.n_elements, dtype=np.int64), (spec.n_tx, 1))
    else:  # centred receive window clipped to the aperture
        half = spec.n_rx // 2
        starts = np.clip(tx - half, 0, spec.n_elements - spec.n_rx)
        rx = starts[:, None] + np.arange(spec.n_rx)[None, :]
    return nodes, tx, rx


def inclusion_phantom(spec: WorkloadSpec, rng: np.random.Generator):
    """(c, rho|None) on the padded grid: inclusions clear of the array row."""
    n, p = spec.n, spec.pml
    c = np.full((n, n), spec.background)
    rho = np.full((n, n), spec.rho0) if spec.density else None
    ix = np.arange(n)[:, None].astype(np.float64)
    iz = np.arange(n)[None, :].astype(np.float64)
    lo_n, hi_n = spec.inclusions
    count = int(rng.integers(lo_n, hi_n + 1))
    for _ in range(count):
        if spec.shape == "disk":
            r = rng.uniform(*spec.radius_cells)
            a = b = r
            ang = 0.0
        else:
            a = rng.uniform(*spec.radius_cells)
            b = rng.uniform(*spec.radius_cells)
            ang = rng.uniform(0.0, np.pi)
        reach = max(a, b)
        cx = rng.uniform(p + reach, p + spec.n_interior - reach)
        cz = rng.uniform(p + 4 + reach, p + spec.n_interior - reach)
        dc = rng.uniform(-spec.contrast, spec.contrast)
        ca, sa = np.cos(ang), np.sin(ang)
        u = (ix - cx) * ca + (iz - cz) * sa
        v = -(ix - cx) * sa + (iz - cz) * ca
        inside = (u / a) ** 2 + (v / b) ** 2 <= 1.0
        c = c + np.where(inside, dc, 0.0)
        if rho is not None:
            rho = np.where(inside, rng.uniform(*spec.rho_range), rho)
    if spec.speckle > 0:
        c = c * (1.0 + spec.speckle * rng.standard_normal((n, n)))
    return c, rho


@dataclass
class Workload:
    spec: WorkloadSpec
    seed: int
    c_true: np.ndarray           # (B, N, N)
    rho: np.ndarray | None       # (B, N, N) or None
    nodes: np.ndarray
    tx: np.ndarray
    rx: np.ndarray
    pulse: np.ndarray
    meta: dict = field(default_factory=dict)


def make_workload(cfg: int | WorkloadSpec, seed: int = 0, n_phantoms: int | None = None) -> Workload:
    spec = cfg if isinstance(cfg, WorkloadSpec) else get_config(cfg)
    B = spec.n_phantoms if n_phantoms is None else int(n_phantoms)
    cs, rhos = [], []
    for b in range(B):
        rng = np.random.default_rng([seed, b])
        c, rho = inclusion_phantom(spec, rng)
        cs.append(c)
        rhos.append(rho)
    nodes, tx, rx = linear_array(spec)
    pulse = gaussian_sine_pulse(spec.f_c, spec.dt, spec.nt)
    rho_arr = np.stack(rhos) if spec.density else None
    return Workload(spec, seed, np.stack(cs), rho_arr, nodes, tx, rx, pulse,
                    meta={"seed": seed, "n_phantoms": B})
