"""Device-resident driver of the DUFWI physics step (plan + workspace + shards).

One :class:`PhysicsEngine` owns a ``libdufwi`` plan for a fixed acquisition
(grid, transmits, receivers, pulse, damping, number of phantoms) and the CUDA
workspace its sweeps need.  Work is organised in *units* — one (phantom,
shot) pair each, ``u = b*S + s`` — processed in contiguous chunks so memory
stays bounded; under ``torch.distributed`` the units are sharded across ranks
(one process per GPU) and the per-rank partial gradients and misfits are
combined with a single ``all_reduce(SUM)`` per gradient evaluation (SURVEY
§8(e)).  Transmissions never interact (forward.py:286-288), so the shard is
exact up to summation order.

PyTorch is only plumbing here: device memory, the current stream and
``torch.distributed``.  Every arithmetic operation on the path runs in the
sm_100a kernels of ``libdufwi.so``.
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._lib import STORE_CHECKPOINT, STORE_FULL, STORE_LAP, STORE_NONE, STORE_STRIPS, check

__all__ = ["PhysicsEngine", "shard_range", "NonFiniteResult", "STORE_NONE", "STORE_FULL",
           "STORE_STRIPS", "STORE_CHECKPOINT", "STORE_LAP"]

_ENGINES = {"auto": _lib.ENGINE_AUTO, "stepwise": _lib.ENGINE_STEPWISE,
            "cluster": _lib.ENGINE_CLUSTER}
#: include/dufwi.h DUFWI_ARITH_*: arithmetic of the sweep kernels
_ARITH = {"f32": 0, "f64": 1}


class NonFiniteResult(FloatingPointError):
    """Raised by the engine when a sweep produced non-finite values."""


def raise_nonfinite(flags) -> None:
    """Raise for host-side flags [traces, gradient] (adjoint.py:75-91 semantics)."""
    if int(flags[0]):
        raise NonFiniteResult("simulation diverged: non-finite receiver samples")
    if int(flags[1]):
        raise NonFiniteResult("gradient blow-up: non-finite accumulated gradient")


def shard_range(n_units: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous block of units for ``rank`` (SURVEY §8(e) partitioning)."""
    base, extra = divmod(n_units, world)
    begin = rank * base + min(rank, extra)
    return begin, begin + base + (1 if rank < extra else 0)


def combine_partials(packed: torch.Tensor) -> None:
    """Sum the per-rank partials — imaging accumulators (B, nx, nz), misfits (B,) and
    the non-finite flag, packed in one f64 buffer — in place: the one collective
    of a gradient evaluation.

    NCCL over NVLink on GPUs; the same call runs on gloo for the CPU tests.
    """
    if not (torch.distributed.is_available() and torch.distributed.is_initialized()):
        return
    if torch.distributed.get_world_size() == 1:
        return
    torch.distributed.all_reduce(packed)


def _ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def _i32(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.int32))


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


@dataclass
class _Workspace:
    mode: int
    units: int
    buf: torch.Tensor


class PhysicsEngine:
    """Forward / adjoint sweeps of the explicit damped 2-D acoustic scheme.

    Parameters mirror the reference's seam ``_propagate(c, d, grid, pulse,
    tx_nodes (P,2), rx_nodes (P,R,2))`` (forward.py:273-281), extended with a
    phantom count ``n_phantoms`` (every phantom uses the same ``S`` shots) and
    an optional density model.
    """

    def __init__(self, *, nx: int, nz: int, nt: int, dx: float, dt: float,
                 tx_nodes, rx_nodes, pulse, element_nodes=None,
                 damping_values=None, damping_profiles=None, n_phantoms: int = 1,
                 has_rho: bool = False, engine: str = "auto", arith: str = "f32", device=None,
                 max_chunk_units: int | None = None, memory_fraction: float = 0.55):
        self._plan = None
        so = _lib.lib()
        if not torch.cuda.is_available():
            raise _lib.ExtensionUnavailable("no CUDA device visible; the DUFWI path is GPU-only")
        self.device = torch.device(device if device is not None else "cuda", )
        if self.device.index is None:
            self.device = torch.device("cuda", torch.cuda.current_device())
        tx = _i32(tx_nodes).reshape(-1, 2)
        rx = _i32(rx_nodes)
        if rx.ndim != 3 or rx.shape[0] != tx.shape[0] or rx.shape[2] != 2:
            raise ValueError("rx_nodes must have shape (S, R, 2) matching tx_nodes (S, 2)")
        el = _i32(element_nodes if element_nodes is not None
                  else np.concatenate([tx, rx.reshape(-1, 2)])).reshape(-1, 2)
        pulse = _f64(pulse)
        if pulse.shape != (nt,):
            raise ValueError("pulse length does not match nt")
        self.nx, self.nz, self.nt, self.dx, self.dt = int(nx), int(nz), int(nt), float(dx), float(dt)
        self.S, self.R, self.B = tx.shape[0], rx.shape[1], int(n_phantoms)
        self.n_units = self.S * self.B
        self.has_rho = bool(has_rho)
        self.engine_kind = engine
        self.tx, self.rx, self.elements, self.pulse = tx, rx, el, pulse
        geo = _lib.Geometry()
        geo.nx, geo.nz, geo.nt = self.nx, self.nz, self.nt
        geo.n_phantoms, geo.n_shots, geo.n_rx, geo.n_elements = self.B, self.S, self.R, el.shape[0]
        geo.has_rho = int(self.has_rho)
        geo.engine = _ENGINES[engine]
        if arith not in _ARITH:
            raise ValueError(f"arith must be one of {sorted(_ARITH)}")
        self.arith = arith
        geo.arith = _ARITH[arith]
        geo.dx, geo.dt = self.dx, self.dt
        keep = [tx, rx, el, pulse]
        I32P, F64P = ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_double)
        geo.tx_host = tx.ctypes.data_as(I32P)
        geo.rx_host = rx.ctypes.data_as(I32P)
        geo.elements_host = el.ctypes.data_as(I32P)
        geo.pulse_host = pulse.ctypes.data_as(F64P)
        if damping_profiles is not None:
            px, pz = _f64(damping_profiles[0]), _f64(damping_profiles[1])
            if px.shape != (self.nx,) or pz.shape != (self.nz,):
                raise ValueError("damping profiles must have shapes (nx,), (nz,)")
            keep += [px, pz]
            geo.px_host = px.ctypes.data_as(F64P)
            geo.pz_host = pz.ctypes.data_as(F64P)
            self.damping = np.maximum(px[:, None], pz[None, :])
        else:
            d = _f64(damping_values if damping_values is not None else np.zeros((self.nx, self.nz)))
            if d.shape != (self.nx, self.nz):
                raise ValueError("damping shape does not match the grid")
            keep.append(d)
            geo.damping_host = d.ctypes.data_as(F64P)
            self.damping = d
        plan = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            check(so.dufwi_plan_create(ctypes.byref(geo), ctypes.byref(plan)))
        self._plan = plan
        self._so = so
        self.max_chunk_units = max_chunk_units
        self.memory_fraction = memory_fraction
        self._ws: dict[int, _Workspace] = {}
        # bumped whenever a workspace is (re)allocated or released: CUDA graphs
        # captured over this engine hold its buffer addresses (unfold.Reconstructor)
        self.ws_generation = 0
        N2 = self.nx * self.nz
        self._flag = torch.zeros(4, dtype=torch.int32, device=self.device)
        self._c = None
        self._rho = None
        self._cluster_path = None
        self._auto_store: dict[bool, int] = {}
        self.box = self._undamped_box()
        # one packed f64 buffer [acc (B*nx*nz) | misfit (B) | flags (1)] so the
        # per-gradient combine across ranks is a single all_reduce
        n_acc = self.B * self.nx * self.nz
        self._red = torch.zeros(n_acc + self.B + 1, dtype=torch.float64, device=self.device)
        self._acc = self._red[:n_acc].view(self.B, self.nx, self.nz)
        self._misfit = self._red[n_acc:n_acc + self.B]
        del N2, keep

    # ------------------------------------------------------------------ misc
    def __del__(self):
        try:
            if self._plan is not None and self._plan.value:
                self._so.dufwi_plan_destroy(self._plan)
        except Exception:  # pragma: no cover - interpreter shutdown
            pass

    @property
    def launch_count(self) -> int:
        return int(self._so.dufwi_plan_launch_count(self._plan))

    @property
    def last_engine(self) -> str:
        code = int(self._so.dufwi_plan_last_engine(self._plan))
        return {1: "stepwise", 2: "cluster"}.get(code, "none")

    def info(self) -> dict:
        """Engine configuration chosen by the plan (cluster shape, shared memory)."""
        buf = (ctypes.c_int64 * 13)()
        n = self._so.dufwi_plan_info(self._plan, buf, 13)
        keys = ("cluster_ok", "cluster_ctas", "rows_per_cta", "rows_per_thread",
                "threads_per_cta", "f64_exchange", "smem_forward", "smem_adjoint",
                "clusters_resident", "adjoint_cluster_ctas", "adjoint_rows_per_thread",
                "adjoint_threads_per_cta", "stepwise_kernels")
        out = {k: int(buf[i]) for i, k in enumerate(keys[:n])}
        if "stepwise_kernels" in out:
            out["stepwise_kernels"] = ("lean", "vec", "stream", "tile")[out["stepwise_kernels"]]
        return out

    def _stream(self) -> int:
        return torch.cuda.current_stream(self.device).cuda_stream

    def _undamped_box(self):
        ix, iz = np.nonzero(self.damping == 0.0)
        if ix.size == 0:
            return None
        box = (ix.min(), ix.max(), iz.min(), iz.max())
        inside = np.zeros_like(self.damping, dtype=bool)
        inside[box[0]:box[1] + 1, box[2]:box[3] + 1] = True
        return box if np.array_equal(inside, self.damping == 0.0) else None

    def local_units(self) -> tuple[int, int]:
        """This rank's unit range (all units without torch.distributed)."""
        if torch.distributed.is_available() and torch.distributed.is_initialized():
            return shard_range(self.n_units, torch.distributed.get_rank(),
                               torch.distributed.get_world_size())
        return 0, self.n_units

    # ------------------------------------------------------------- model
    def set_model(self, c, rho=None) -> None:
        """Speed map(s) (B, nx, nz) or (nx, nz); density likewise when has_rho."""
        c_t = self._as_dev(c, torch.float64).reshape(self.B, self.nx, self.nz).contiguous()
        rho_t = None
        if self.has_rho:
            if rho is None:
                raise ValueError("engine was built for a density model; pass rho")
            rho_t = self._as_dev(rho, torch.float64).reshape(self.B, self.nx, self.nz).contiguous()
        self._c, self._rho = c_t, rho_t
        check(self._so.dufwi_set_model(self._plan, _ptr(c_t), _ptr(rho_t), self._stream()))

    def _as_dev(self, a, dtype) -> torch.Tensor:
        if isinstance(a, torch.Tensor):
            return a.to(device=self.device, dtype=dtype)
        return torch.as_tensor(np.array(a, copy=True), dtype=dtype).to(self.device, non_blocking=False)

    # --------------------------------------------------------- workspace
    def _ws_bytes(self, mode: int, units: int) -> int:
        out = ctypes.c_size_t()
        check(self._so.dufwi_workspace_bytes(self._plan, mode, units, ctypes.byref(out)))
        return int(out.value)

    def chunk_units(self, mode: int, n: int) -> int:
        if self.max_chunk_units:
            return max(1, min(n, self.max_chunk_units))
        ws = self._ws.get(mode)
        if ws is not None and ws.buf.numel() >= self._ws_bytes(mode, n):
            return n  # the held workspace already fits: no device query on the hot path
        free, _ = torch.cuda.mem_get_info(self.device)
        held = sum(w.buf.numel() for w in self._ws.values())
        budget = (free + held) * self.memory_fraction
        per = self._ws_bytes(mode, 1)
        u = int(max(1, min(n, budget // max(per, 1))))
        while u > 1 and self._ws_bytes(mode, u) > budget:
            u = max(1, int(u * 0.8))
        return u

    def _workspace(self, mode: int, units: int) -> _Workspace:
        ws = self._ws.get(mode)
        need = self._ws_bytes(mode, units)
        if ws is None or ws.buf.numel() < need:
            self._ws.pop(mode, None)
            ws = _Workspace(mode, units, torch.empty(need, dtype=torch.uint8, device=self.device))
            self._ws[mode] = ws
            self.ws_generation += 1
        return ws

    def reserve(self, store: str = "auto", mask: bool = True,
                units: tuple[int, int] | None = None) -> int:
        """Allocate the workspace a gradient over ``units`` (default: this rank's
        shard) will use, outside any timed region; returns the chunk size."""
        u0, u1 = units if units is not None else self.local_units()
        mode = self.pick_store(mask, store)
        chunk = self.chunk_units(mode, max(u1 - u0, 1))
        self._workspace(mode, chunk)
        return chunk

    def release_workspace(self) -> None:
        self._ws.clear()
        self.ws_generation += 1

    # ----------------------------------------------------------- sweeps
    def _require_model(self):
        if self._c is None:
            raise RuntimeError("set_model() must be called before a sweep")

    def forward(self, units: tuple[int, int] | None = None, check_finite: bool = True) -> torch.Tensor:
        """Receiver traces (U, R, nt) f32 for units [begin, end) — forward.py:273-313."""
        self._require_model()
        u0, u1 = units if units is not None else (0, self.n_units)
        n = u1 - u0
        out = torch.empty((n, self.R, self.nt), dtype=torch.float32, device=self.device)
        chunk = self.chunk_units(STORE_NONE, n)
        ws = self._workspace(STORE_NONE, chunk)
        self._flag.zero_()
        st = self._stream()
        for a in range(u0, u1, chunk):
            U = min(chunk, u1 - a)
            check(self._so.dufwi_forward(self._plan, STORE_NONE, a, U, _ptr(out[a - u0:]),
                                         _ptr(self._flag), _ptr(ws.buf), ws.buf.numel(), st))
        if check_finite and int(self._flag[0].item()):
            raise NonFiniteResult("simulation diverged: non-finite receiver samples")
        return out

    def wavefield_history(self, unit: int = 0) -> torch.Tensor:
        """Full f32 history (nt, nx, nz) of one unit (simulate_wavefield, forward.py:316-332)."""
        self._require_model()
        ws = self._workspace(STORE_FULL, 1)
        check(self._so.dufwi_forward(self._plan, STORE_FULL, unit, 1, None, _ptr(self._flag),
                                     _ptr(ws.buf), ws.buf.numel(), self._stream()))
        off = ctypes.c_size_t()
        check(self._so.dufwi_history_offset(self._plan, 1, ctypes.byref(off)))
        n = self.nt * self.nx * self.nz
        flat = ws.buf[off.value: off.value + 4 * n].view(torch.float32)
        return flat.view(self.nt, self.nx, self.nz).clone()

    @property
    def cluster_path(self) -> bool:
        """The sweeps run on the cluster engine (the grid fits, not forced stepwise)."""
        if self._cluster_path is None:
            self._cluster_path = bool(self.info().get("cluster_ok")) and self.engine_kind != "stepwise"
        return self._cluster_path

    def pick_store(self, mask: bool, store: str = "auto") -> int:
        """Forward-history strategy of a gradient: "full" f32 history, "strips"
        (1-cell ring of the undamped box + backward reconstruction),
        "checkpoint" (snapshots + segment recomputation, any damping), "lap"
        (cluster engine: the forward stores the imaging operand L(u), the
        adjoint carries only lam) or "auto": lap on the cluster engine when a
        wave of units fits the memory budget, else strips where they apply,
        else full history when one unit's fits, else checkpointing."""
        if store == "full":
            return STORE_FULL
        if store == "checkpoint":
            return STORE_CHECKPOINT
        if store == "lap":
            if not self.cluster_path:
                raise ValueError("L(u) history storage needs the cluster engine")
            if self.box is None or (not mask and self.box != (0, self.nx - 1, 0, self.nz - 1)):
                raise ValueError("L(u) history storage images the undamped box; use mask=True")
            if self.nz % 4:
                raise ValueError("L(u) history storage needs nz % 4 == 0")
            return STORE_LAP
        if store == "strips":
            if self.box is None:
                raise ValueError("strip storage needs a rectangular undamped box")
            if not mask and self.box != (0, self.nx - 1, 0, self.nz - 1):
                raise ValueError("strip storage only reconstructs the undamped box; use mask=True")
            return STORE_STRIPS
        if store != "auto":
            raise ValueError(f"unknown store {store!r}")
        # decided once per mask setting: no device query inside captured CUDA graphs
        hit = self._auto_store.get(bool(mask))
        if hit is not None:
            return hit
        self._auto_store[bool(mask)] = mode = self._auto_pick(mask)
        return mode

    def _auto_pick(self, mask: bool) -> int:
        free, _ = torch.cuda.mem_get_info(self.device)
        held = sum(w.buf.numel() for w in self._ws.values())
        box_ok = self.box is not None and (mask or self.box == (0, self.nx - 1, 0, self.nz - 1))
        if (self.cluster_path and box_ok and self.nz % 4 == 0
                and os.environ.get("DUFWI_LAP", "1") != "0"):
            wave = min(self.n_units, 16)
            if self._ws_bytes(STORE_LAP, wave) <= (free + held) * self.memory_fraction:
                return STORE_LAP
        if self.box is not None and (mask or self.box == (0, self.nx - 1, 0, self.nz - 1)):
            return STORE_STRIPS
        if self._ws_bytes(STORE_FULL, 1) > (free + held) * self.memory_fraction:
            return STORE_CHECKPOINT
        return STORE_FULL

    def misfit_and_gradient(self, obs: torch.Tensor, *, mask: bool = True, guard_radius: int = 2,
                            store: str = "auto", units: tuple[int, int] | None = None,
                            reduce: bool = True, check_finite: bool = True,
                            return_traces: bool = False):
        """Per-phantom misfit (B,) and SoS gradient (B, nx, nz), both f64 on device.

        ``obs`` is the observed data for all units, (B*S, R, nt) f64 on device
        (the ChannelData layout of grid.py:164-183, phantoms stacked).
        Under torch.distributed, and only when ``units`` is None, the call is a
        collective: the unit range is this rank's shard and the partial sums are
        all-reduced (``reduce``) before the mask/scaling epilogue.  An explicit
        ``units`` range is a local computation on every rank.
        """
        self._require_model()
        self._check_obs(obs)
        dist = torch.distributed.is_available() and torch.distributed.is_initialized()
        collective = dist and units is None
        u0, u1 = units if units is not None else self.local_units()
        mode = self.pick_store(mask, store)
        n = u1 - u0
        chunk = self.chunk_units(mode, max(n, 1))
        ws = self._workspace(mode, chunk) if n > 0 else None
        st = self._stream()
        self._red.zero_()
        self._flag.zero_()
        traces =torch.empty((max(n, 0), self.R, self.nt), dtype=torch.float32, device=self.device)
        if obs.dtype != torch.float64 or obs.device != self.device:
            obs = obs.to(self.device, torch.float64)
        obs = obs.contiguous()
        for a in range(u0, u1, chunk):
            U = min(chunk, u1 - a)
            tr = traces[a - u0:]
            check(self._so.dufwi_forward(self._plan, mode, a, U, _ptr(tr), _ptr(self._flag),
                                         _ptr(ws.buf), ws.buf.numel(), st))
            check(self._so.dufwi_residual(self._plan, a, U, _ptr(tr), _ptr(obs[a:]),
                                          _ptr(self._misfit), _ptr(ws.buf), ws.buf.numel(), st))
            check(self._so.dufwi_adjoint(self._plan, mode, a, U, _ptr(ws.buf), ws.buf.numel(),
                                         _ptr(self._acc), st))
        if collective and reduce:
            self._red[-1] = self._flag[0].double()
            combine_partials(self._red)
            self._flag[0] = (self._red[-1] > 0).int()
        grad = torch.empty_like(self._acc)
        check(self._so.dufwi_finalize_gradient(self._plan, _ptr(self._acc), int(bool(mask)),
                                               int(guard_radius), _ptr(grad),
                                               _ptr(self._flag[1:]), st))
        if check_finite:
            raise_nonfinite(self._flag.cpu())
        misfit = self._misfit.clone()
        if return_traces:
            return misfit, grad, traces
        return misfit, grad

    def _check_obs(self, obs) -> None:
        """Observed data must cover every unit: (B*S, R, nt) (grid.py:164-183 per phantom)."""
        want = (self.n_units, self.R, self.nt)
        if tuple(obs.shape) != want:
            raise ValueError(f"observed data shape {tuple(obs.shape)} != (units, R, nt) {want}")

    def misfit(self, obs: torch.Tensor, units: tuple[int, int] | None = None,
               check_finite: bool = True) -> torch.Tensor:
        """Per-phantom misfit sum((traces - obs)^2) (B,) f64 of a forward sweep alone
        (data_misfit of simulate_all, adjoint.py:67-72); local, never a collective."""
        self._require_model()
        self._check_obs(obs)
        u0, u1 = units if units is not None else (0, self.n_units)
        n = u1 - u0
        chunk = self.chunk_units(STORE_NONE, n)
        ws = self._workspace(STORE_NONE, chunk)
        st = self._stream()
        self._flag.zero_()
        mis = torch.zeros(self.B, dtype=torch.float64, device=self.device)
        tr = torch.empty((chunk, self.R, self.nt), dtype=torch.float32, device=self.device)
        obs = obs.to(self.device, torch.float64).contiguous()
        for a in range(u0, u1, chunk):
            U = min(chunk, u1 - a)
            check(self._so.dufwi_forward(self._plan, STORE_NONE, a, U, _ptr(tr), _ptr(self._flag),
                                         _ptr(ws.buf), ws.buf.numel(), st))
            check(self._so.dufwi_residual(self._plan, a, U, _ptr(tr), _ptr(obs[a:]), _ptr(mis),
                                          _ptr(ws.buf), ws.buf.numel(), st))
        if check_finite and int(self._flag[0].item()):
            raise NonFiniteResult("simulation diverged: non-finite receiver samples")
        return mis

    def last_flags(self) -> torch.Tensor:
        """Device copy of the last call's non-finite flags [traces, gradient] (no sync);
        pass to :func:`raise_nonfinite` after a host sync to check deferred results."""
        return self._flag[:2].clone()

    # ------------------------------------------------------------ timing
    def time_sweeps(self, obs: torch.Tensor, reps: int = 3, mask: bool = True,
                    store: str = "auto", units: tuple[int, int] | None = None) -> dict:
        """Average CUDA-event time of one forward and one adjoint C-ABI call over this
        rank's units (one chunk), on the launching stream — the roofline denominators."""
        self._require_model()
        self._check_obs(obs)
        u0, u1 = units if units is not None else self.local_units()
        mode = self.pick_store(mask, store)
        U = u1 - u0
        ws = self._workspace(mode, U)
        st = self._stream()
        acc = torch.zeros_like(self._acc)
        mis = torch.zeros_like(self._misfit)
        tr = torch.empty((U, self.R, self.nt), dtype=torch.float32, device=self.device)
        obs = obs.to(self.device, torch.float64).contiguous()
        ev = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(reps + 1)]
        for r in range(reps + 1):
            ev[r][0].record()
            check(self._so.dufwi_forward(self._plan, mode, u0, U, _ptr(tr), _ptr(self._flag),
                                         _ptr(ws.buf), ws.buf.numel(), st))
            ev[r][1].record()
            check(self._so.dufwi_residual(self._plan, u0, U, _ptr(tr), _ptr(obs[u0:]), _ptr(mis),
                                          _ptr(ws.buf), ws.buf.numel(), st))
            ev[r][2].record()
            check(self._so.dufwi_adjoint(self._plan, mode, u0, U, _ptr(ws.buf), ws.buf.numel(),
                                         _ptr(acc), st))
            ev[r][3].record()
        torch.cuda.synchronize(self.device)
        f = [ev[r][0].elapsed_time(ev[r][1]) for r in range(1, reps + 1)]
        a = [ev[r][2].elapsed_time(ev[r][3]) for r in range(1, reps + 1)]
        return {"units": U, "forward_ms": sum(f) / reps, "adjoint_ms": sum(a) / reps,
                "store": {STORE_FULL: "full", STORE_STRIPS: "strips", STORE_LAP: "lap",
                          STORE_CHECKPOINT: "checkpoint"}.get(mode, "none"),
                "engine": self.last_engine}
