"""ctypes binding of ``libdufwi.so`` (the C ABI declared in ``include/dufwi.h``).

The shared library is built in-tree by ``__graft_entry__.build()`` (nvcc,
``-gencode arch=compute_100a,code=sm_100a``).  There is no fallback: if the
library is missing or no CUDA device is visible, every compute entry point
raises :class:`ExtensionUnavailable`.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

__all__ = ["LIB_PATH", "ExtensionUnavailable", "DufwiError", "Geometry", "lib", "check",
           "EXPORTED_SYMBOLS", "STORE_NONE", "STORE_FULL", "STORE_STRIPS", "STORE_CHECKPOINT", "STORE_LAP",
           "ENGINE_AUTO", "ENGINE_STEPWISE", "ENGINE_CLUSTER"]

LIB_PATH = Path(os.environ.get("DUFWI_LIB", Path(__file__).resolve().parent / "libdufwi.so"))

STORE_NONE, STORE_FULL, STORE_STRIPS, STORE_CHECKPOINT, STORE_LAP = 0, 1, 2, 3, 4
ENGINE_AUTO, ENGINE_STEPWISE, ENGINE_CLUSTER = 0, 1, 2

EXPORTED_SYMBOLS = (
    "dufwi_plan_create", "dufwi_plan_destroy", "dufwi_set_model", "dufwi_workspace_bytes",
    "dufwi_forward", "dufwi_history_offset", "dufwi_residual", "dufwi_adjoint",
    "dufwi_finalize_gradient", "dufwi_plan_launch_count", "dufwi_plan_last_engine", "dufwi_plan_info", "dufwi_last_error", "dufwi_version",
    "dufwi_net_input", "dufwi_apply_update", "dufwi_laplacian", "dufwi_step_field",
)


# plan-less library kernels launched (the update-net glue: dufwi_net_input = 2,
# dufwi_apply_update = 1), for launch-count evidence next to the plans' counters
GLUE_LAUNCHES = [0]


class ExtensionUnavailable(RuntimeError):
    """libdufwi.so is not built/loadable or no CUDA device is present."""


class DufwiError(RuntimeError):
    """A C-ABI call returned a non-zero status."""

    def __init__(self, code: int, message: str):
        super().__init__(f"dufwi error {code}: {message}")
        self.code = code


class Geometry(ctypes.Structure):
    """Mirror of ``dufwi_geometry_t``."""

    _fields_ = [
        ("nx", ctypes.c_int32), ("nz", ctypes.c_int32), ("nt", ctypes.c_int32),
        ("n_phantoms", ctypes.c_int32), ("n_shots", ctypes.c_int32), ("n_rx", ctypes.c_int32),
        ("n_elements", ctypes.c_int32), ("has_rho", ctypes.c_int32), ("engine", ctypes.c_int32),
        ("arith", ctypes.c_int32),
        ("dx", ctypes.c_double), ("dt", ctypes.c_double),
        ("tx_host", ctypes.POINTER(ctypes.c_int32)),
        ("rx_host", ctypes.POINTER(ctypes.c_int32)),
        ("elements_host", ctypes.POINTER(ctypes.c_int32)),
        ("px_host", ctypes.POINTER(ctypes.c_double)),
        ("pz_host", ctypes.POINTER(ctypes.c_double)),
        ("damping_host", ctypes.POINTER(ctypes.c_double)),
        ("pulse_host", ctypes.POINTER(ctypes.c_double)),
    ]


_LIB = None


def _declare(so: ctypes.CDLL) -> None:
    vp, i32, i64, sz = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_size_t
    so.dufwi_plan_create.argtypes = [ctypes.POINTER(Geometry), ctypes.POINTER(vp)]
    so.dufwi_plan_destroy.argtypes = [vp]
    so.dufwi_set_model.argtypes = [vp, vp, vp, vp]
    so.dufwi_workspace_bytes.argtypes = [vp, i32, i32, ctypes.POINTER(sz)]
    so.dufwi_forward.argtypes = [vp, i32, i32, i32, vp, vp, vp, sz, vp]
    so.dufwi_history_offset.argtypes = [vp, i32, ctypes.POINTER(sz)]
    so.dufwi_residual.argtypes = [vp, i32, i32, vp, vp, vp, vp, sz, vp]
    so.dufwi_adjoint.argtypes = [vp, i32, i32, i32, vp, sz, vp, vp]
    so.dufwi_finalize_gradient.argtypes = [vp, vp, i32, i32, vp, vp, vp]
    so.dufwi_plan_launch_count.argtypes = [vp]
    so.dufwi_plan_launch_count.restype = i64
    so.dufwi_plan_last_engine.argtypes = [vp]
    so.dufwi_plan_last_engine.restype = i32
    so.dufwi_plan_info.argtypes = [vp, ctypes.POINTER(i64), i32]
    so.dufwi_plan_info.restype = i32
    f64 = ctypes.c_double
    so.dufwi_net_input.argtypes = [vp, vp, i32, i64, f64, f64, vp, vp, vp]
    so.dufwi_apply_update.argtypes = [vp, vp, i64, f64, f64, f64, vp, vp]
    so.dufwi_laplacian.argtypes = [vp, i64, i32, i32, f64, vp, vp]
    so.dufwi_step_field.argtypes = [vp, vp, vp, vp, vp, i32, i32, f64, f64, vp, vp]
    so.dufwi_last_error.restype = ctypes.c_char_p
    so.dufwi_version.restype = ctypes.c_char_p
    for name in ("dufwi_plan_create", "dufwi_plan_destroy", "dufwi_set_model",
                 "dufwi_workspace_bytes", "dufwi_forward", "dufwi_history_offset", "dufwi_residual",
                 "dufwi_adjoint", "dufwi_finalize_gradient", "dufwi_net_input",
                 "dufwi_apply_update", "dufwi_laplacian", "dufwi_step_field"):
        getattr(so, name).restype = ctypes.c_int


def lib() -> ctypes.CDLL:
    """Load libdufwi.so once; raise loudly if it is absent."""
    global _LIB
    if _LIB is None:
        if not LIB_PATH.exists():
            raise ExtensionUnavailable(
                f"{LIB_PATH} not built — run `python -c 'import __graft_entry__ as g; g.build()'`")
        try:
            so = ctypes.CDLL(str(LIB_PATH), mode=os.RTLD_NOW | getattr(os, "RTLD_GLOBAL", 0))
        except OSError as exc:  # pragma: no cover - environment dependent
            raise ExtensionUnavailable(f"cannot load {LIB_PATH}: {exc}") from exc
        _declare(so)
        _LIB = so
    return _LIB


def check(rc: int) -> None:
    if rc != 0:
        msg = lib().dufwi_last_error().decode(errors="replace")
        raise DufwiError(rc, msg)
