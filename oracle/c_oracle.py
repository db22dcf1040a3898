"""TEST INFRASTRUCTURE — ctypes front end of the C float64 checker (``dufwi_oracle_c.c``).

Same signatures and results as :mod:`oracle.dufwi_oracle` (``forward_sweep``,
``misfit_gradient``, ``unfold_reconstruct``), restating the same reference code
(forward.py:211-313, adjoint.py:94-138, unfold.py:253-267), but multi-threaded
over transmissions and with f64 snapshot checkpointing instead of the full
field history — the sizes of BASELINE.json configs 2-4 (a full f64 history is
10 GB per shot at config 3 and 57 GB at config 4) stay in a few GB.

The coefficient maps (A, B, E, dE/dc, density face weights) and the residual
misfit are computed here with the NumPy restatement's own expressions, so only
the per-step stencil arithmetic runs in C.  ``tests/test_c_oracle.py`` pins it
against the NumPy restatement (traces bit-identical; gradients to 1e-13, the
shot-summation order differs) and, through it, the reference fixtures.
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess
from pathlib import Path

import numpy as np

from . import dufwi_oracle as _np_oracle

__all__ = ["available", "build", "forward_sweep", "misfit_gradient", "unfold_reconstruct",
           "default_threads", "LIB"]

HERE = Path(__file__).resolve().parent
LIB = HERE / "_build" / "libdufwi_oracle.so"
_SO = None


def build(force: bool = False) -> Path:
    """Compile the checker with gcc (oracle/Makefile); cheap no-op when up to date."""
    src = HERE / "dufwi_oracle_c.c"
    if force or not LIB.exists() or LIB.stat().st_mtime < src.stat().st_mtime:
        subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
    return LIB


def available() -> bool:
    try:
        _lib()
        return True
    except Exception:
        return False


def _lib():
    global _SO
    if _SO is None:
        if not LIB.exists():
            build()
        so = ctypes.CDLL(str(LIB))
        P = ctypes.c_void_p
        i32, f64 = ctypes.c_int, ctypes.c_double
        so.dufwi_oracle_forward.argtypes = [i32, i32, i32, f64, P, P, P, P, P, i32, P, i32, P, P, i32]
        so.dufwi_oracle_gradient.argtypes = [i32, i32, i32, f64, P, P, P, P, P, i32, P, i32, P, P,
                                             P, P, i32, i32]
        so.dufwi_oracle_forward.restype = i32
        so.dufwi_oracle_gradient.restype = i32
        _SO = so
    return _SO


def default_threads() -> int:
    try:
        return max(1, len(os.sched_getaffinity(0)))
    except AttributeError:  # pragma: no cover
        return max(1, os.cpu_count() or 1)


def _p(a: np.ndarray | None):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _model(c, d, dx, dt, pulse, rho):
    c = np.ascontiguousarray(c, dtype=np.float64)
    d = np.ascontiguousarray(d, dtype=np.float64)
    A, B, E = (np.ascontiguousarray(x) for x in _np_oracle.step_coeffs(c, d, dt))
    w = None
    if rho is not None:
        w = np.ascontiguousarray(np.stack(_np_oracle.rho_face_weights(
            np.asarray(rho, dtype=np.float64))))
    pulse = np.ascontiguousarray(pulse, dtype=np.float64)
    return c, d, A, B, E, w, pulse


def forward_sweep(c, d, dx, dt, pulse, tx, rx, rho=None, threads: int | None = None):
    """Receiver traces (P, R, nt) — same values as ``oracle.forward_sweep`` (bit-identical)."""
    c, d, A, B, E, w, pulse = _model(c, d, dx, dt, pulse, rho)
    nx, nz = c.shape
    nt = pulse.shape[0]
    tx = np.ascontiguousarray(tx, dtype=np.int32).reshape(-1, 2)
    rx = np.ascontiguousarray(rx, dtype=np.int32)
    P, R = rx.shape[0], rx.shape[1]
    tr = np.empty((P, R, nt))
    rc = _lib().dufwi_oracle_forward(nx, nz, nt, float(dx), _p(A), _p(B), _p(E), _p(w), _p(pulse),
                                     P, _p(tx), R, _p(rx), _p(tr), threads or default_threads())
    if rc:
        raise FloatingPointError("simulation diverged: non-finite receiver samples")
    return tr, None


def default_segment(nt: int) -> int:
    """Checkpoint interval minimising snapshots (2 fields each) + one segment's history."""
    return max(2, int(math.ceil(math.sqrt(2.0 * nt))))


def misfit_gradient(c, d, dx, dt, pulse, tx, rx, obs, element_nodes=None, mask=True,
                    guard_radius=2, rho=None, threads: int | None = None, seg: int | None = None,
                    return_parts: bool = False):
    """Misfit, gradient and traces, as ``oracle.misfit_gradient`` (adjoint.py:94-138)."""
    c, d, A, B, E, w, pulse = _model(c, d, dx, dt, pulse, rho)
    nx, nz = c.shape
    nt = pulse.shape[0]
    tx = np.ascontiguousarray(tx, dtype=np.int32).reshape(-1, 2)
    rx = np.ascontiguousarray(rx, dtype=np.int32)
    P, R = rx.shape[0], rx.shape[1]
    obs = np.ascontiguousarray(obs, dtype=np.float64)
    if obs.shape != (P, R, nt):
        raise ValueError(f"obs shape {obs.shape} != {(P, R, nt)}")
    tr = np.empty((P, R, nt))
    img = np.empty((P, nx, nz))
    rc = _lib().dufwi_oracle_gradient(nx, nz, nt, float(dx), _p(A), _p(B), _p(E), _p(w),
                                      _p(pulse), P, _p(tx), R, _p(rx), _p(obs), _p(tr), _p(img),
                                      int(seg or default_segment(nt)), threads or default_threads())
    if rc:
        if not np.all(np.isfinite(tr)):
            raise FloatingPointError("simulation diverged: non-finite receiver samples")
        raise FloatingPointError("gradient blow-up")
    diff = tr - obs
    misfit = float(np.sum(diff ** 2))  # adjoint.py:114, the NumPy expression
    dEdc = 2.0 * c * dt ** 2 / (1.0 + d * dt)  # adjoint.py:117
    acc = np.zeros((nx, nz))
    for p in range(P):  # shot order
        acc += img[p]
    grad = dEdc * acc
    if mask:
        nodes = element_nodes if element_nodes is not None else np.concatenate(
            [tx.reshape(-1, 2), rx.reshape(-1, 2)])
        grad = np.where(_np_oracle.guard_mask(d, nodes, guard_radius), grad, 0.0)
    if return_parts:
        return misfit, grad, tr, img
    return misfit, grad, tr


def unfold_reconstruct(obs, c0, predict_updates, bounds, d, dx, dt, pulse, tx, rx,
                       element_nodes=None, rho=None, guard_radius=2, threads=None):
    """K-stage unfolded inference (unfold.py:253-267), as ``oracle.unfold_reconstruct``."""
    lo, hi = bounds
    c = np.clip(np.asarray(c0, dtype=np.float64), lo, hi)
    maps, grads = [], []
    for f in predict_updates:
        _, g, _ = misfit_gradient(c, d, dx, dt, pulse, tx, rx, obs, element_nodes,
                                  rho=rho, guard_radius=guard_radius, threads=threads)
        grads.append(g)
        c = np.clip(c + f(c, g), lo, hi)
        maps.append(c)
    return maps, grads
