"""B200-native DUFWI physics step (drop-in for the hot path of fwilab).

Public API mirrors the reference package's forward / gradient / unfolded
inference entry points.  Importing the package never touches the GPU; the
first sweep loads ``libdufwi.so`` and fails loudly if it is missing.
"""

__version__ = "0.1.0"

from .grid import (SOS_LIMIT, AcquisitionGeometry, ChannelData, CflCheck, DensityMap,
                   GeometryError, Grid2D, SosMap, build_geometry, check_cfl, homogeneous_map,
                   linear_geometry)
from .forward import (DampingProfile, NumericError, SourcePulse, Wavefield, build_pml, laplacian,
                      make_source_pulse, simulate_all, simulate_transmission, simulate_wavefield,
                      step_wavefield, zero_damping)
from .adjoint import (GradientMap, compute_gradient, data_misfit, fd_gradient_oracle,
                      gradient_mask, misfit_and_gradient, misfit_and_gradient_batch)
from .unfold import (InversionSetup, Reconstructor, cfl_safe_bounds, clamp_sos, unfold_infer,
                     unfold_infer_batch)
from ._lib import DufwiError, ExtensionUnavailable

__all__ = [
    "AcquisitionGeometry", "ChannelData", "CflCheck", "DensityMap", "GeometryError", "Grid2D",
    "SosMap", "SOS_LIMIT", "build_geometry", "check_cfl", "homogeneous_map", "linear_geometry",
    "DampingProfile", "NumericError", "SourcePulse", "Wavefield", "build_pml", "laplacian",
    "make_source_pulse", "simulate_all", "simulate_transmission", "simulate_wavefield",
    "step_wavefield", "zero_damping", "GradientMap", "compute_gradient", "data_misfit",
    "fd_gradient_oracle", "gradient_mask",
    "misfit_and_gradient", "misfit_and_gradient_batch", "InversionSetup", "Reconstructor",
    "cfl_safe_bounds", "clamp_sos", "unfold_infer", "unfold_infer_batch", "DufwiError", "ExtensionUnavailable",
]
