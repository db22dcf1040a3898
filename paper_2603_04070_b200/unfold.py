"""Unfolded (DUFWI) inference driver — mirror of ``fwilab.unfold`` inference side.

``unfold_infer`` keeps the reference signature (unfold.py:253-267): start from
the clamped initial map, then per stage compute the gradient, apply the
stage network's update and clamp.  The loop is device-resident: the speed
map, gradient and network update never leave the GPU between stages; the
returned :class:`SosMap` list is copied to the host once at the end.
"""

from __future__ import annotations

import os
from dataclasses import dataclass, field

import numpy as np

from .forward import DampingProfile, NumericError, SourcePulse, _check_simulation_inputs, get_engine, zero_damping
from .grid import ChannelData, Grid2D, SosMap, check_cfl
from .network import NormSpec

__all__ = ["InversionSetup", "cfl_safe_bounds", "clamp_sos", "unfold_infer", "unfold_infer_batch",
           "Reconstructor"]


@dataclass(frozen=True)
class InversionSetup:
    """Physics context of training and inference (unfold.py:66-74); ``density``
    is an extension."""

    pulse: SourcePulse
    damping: DampingProfile | None = None
    bounds: tuple[float, float] = (1300.0, 3200.0)
    water_speed: float = 1500.0
    norm: NormSpec = field(default_factory=NormSpec)
    density: np.ndarray | None = None


def cfl_safe_bounds(grid: Grid2D, bounds: tuple[float, float], safety: float = 0.999):
    """Cap the upper bound at the stability limit (unfold.py:117-131)."""
    limit = safety * grid.dx / (grid.dt * np.sqrt(2.0))
    lo, hi = bounds
    if lo >= limit:
        raise ValueError(f"lower bound {lo} m/s already exceeds the CFL limit {limit:.1f} m/s")
    return (lo, min(hi, limit))


def clamp_sos(sos: SosMap, bounds: tuple[float, float]) -> SosMap:
    """Elementwise clamp, idempotent (unfold.py:134-142)."""
    lo, hi = bounds
    if not lo < hi:
        raise ValueError("bounds must satisfy c_min < c_max")
    v = np.clip(sos.values, lo, hi)
    return sos if np.array_equal(v, sos.values) else sos.with_values(v)


class Reconstructor:
    """Device-resident K-stage unfolded inference for B phantoms sharing an acquisition.

    ``reconstruct(obs, c0)`` takes device tensors ((B*S, R, nt) f64 observed
    data and (B, nx, nz) initial maps) and returns the list of stage maps
    (B, nx, nz) on device, plus the per-stage gradients when asked.

    In a single process the K stages (sweeps, residual, epilogue, networks,
    clamps: ~30 launches per stage) are captured into a CUDA graph on the
    second call with the same shapes and replayed from then on; the inputs are
    copied into the graph's static buffers first.  The first call, calls under
    torch.distributed, with host networks or when gradients are kept launch the
    stages eagerly.
    """

    def __init__(self, engine, nets, bounds, guard_radius: int = 2, rho=None,
                 graph: bool | None = None, collective: bool = True, cfl_grid=None):
        self.engine = engine
        self.nets = list(nets)
        self.bounds = bounds
        self.guard_radius = guard_radius
        self.rho = rho
        # collective=False: every rank computes all units of its own call (the
        # per-sample public API); True: units sharded across torch.distributed ranks
        self.collective = collective
        # when the upper clamp bound exceeds the CFL limit of this grid, each
        # stage's input maximum is recorded on the device and checked after the
        # sync, raising the reference's ValueError (forward.py:259-263 runs in
        # every stage's compute_gradient, adjoint.py:105)
        self.cfl_grid = None
        if cfl_grid is not None and not check_cfl(cfl_grid, bounds[1]).ok:
            self.cfl_grid = cfl_grid
        # DUFWI_GRAPH=0 launches the stages eagerly (A/B timing, debugging)
        self.graph = (os.environ.get("DUFWI_GRAPH", "1") != "0") if graph is None else graph
        self._g = None  # (key, graph, static obs, static c0, maps, flags, launches, ws generation)
        self._seen = None  # key of the last eager call (capture on the next one)
        self.replayed_launches = 0

    def _update(self, net, c, g):
        """clamp(c + update(c, g)) of one stage for the phantoms in ``c`` (unfold.py:263-265)."""
        import torch

        lo, hi = self.bounds
        if hasattr(net, "stage_device") and c.is_cuda:
            return net.stage_device(c, g, lo, hi)  # normalisation + update in libdufwi
        if hasattr(net, "predict_update_device"):
            return torch.clamp(c + net.predict_update_device(c, g), lo, hi)
        # a host network (e.g. the reference's NumPy CNN): one round trip per stage
        upd = torch.stack([torch.as_tensor(net.predict_update(ci.cpu().numpy(), gi.cpu().numpy()))
                           for ci, gi in zip(c, g)]).to(c.device)
        return torch.clamp(c + upd, lo, hi)

    def _stages(self, obs, c0, keep_gradients: bool, check_finite: bool):
        import torch

        from .engine import raise_nonfinite, shard_range

        lo, hi = self.bounds
        c = torch.clamp(c0.to(torch.float64), lo, hi)
        maps, grads, flags, cmax = [], [], [], []
        dist = (self.collective and torch.distributed.is_available()
                and torch.distributed.is_initialized() and torch.distributed.get_world_size() > 1)
        units = None if self.collective else (0, self.engine.n_units)
        for net in self.nets:
            if self.cfl_grid is not None:
                cmax.append(c.amax().reshape(1))
            self.engine.set_model(c, self.rho)
            # non-finite checks are deferred to one host sync after the last stage,
            # so the stages queue back to back on the device
            _, g = self.engine.misfit_and_gradient(obs, guard_radius=self.guard_radius,
                                                   check_finite=False, units=units)
            flags.append(self.engine.last_flags())
            if check_finite and not hasattr(net, "predict_update_device"):
                # a host network reads the gradient now: check before handing it over
                # (the flags are part of the combined partials: every rank raises alike)
                raise_nonfinite(flags[-1].cpu())
            if dist:
                # each phantom's update runs on ONE rank (phantoms split like units,
                # engine.shard_range), the others contribute exact zeros to one
                # all_reduce: no replicated network work (weak scaling keeps the
                # per-rank network cost of one process), and every rank holds the same
                # bits whatever cuDNN algorithm each rank would have picked
                b0, b1 = shard_range(c.shape[0], torch.distributed.get_rank(),
                                     torch.distributed.get_world_size())
                nxt = torch.zeros_like(c)
                if b1 > b0:
                    nxt[b0:b1] = self._update(net, c[b0:b1], g[b0:b1])
                torch.distributed.all_reduce(nxt)
                c = nxt
            else:
                c = self._update(net, c, g)
            maps.append(c)
            if keep_gradients:
                grads.append(g)
        stage_cmax = torch.cat(cmax) if cmax else None
        return maps, grads, torch.stack(flags), stage_cmax

    def _check_stages(self, flags, stage_cmax) -> None:
        """Raise for the first failing stage, in the reference's order: the CFL check of
        the stage input (forward.py:259-263), then the non-finite checks."""
        from .engine import raise_nonfinite

        cm = stage_cmax.cpu().tolist() if stage_cmax is not None else None
        for k, f in enumerate(flags.cpu()):
            if cm is not None:
                cfl = check_cfl(self.cfl_grid, cm[k])
                if not cfl.ok:
                    raise ValueError(f"CFL violated: ratio {cfl.ratio:.4f} > 1 for c_max={cm[k]} m/s")
            raise_nonfinite(f)

    def _graphable(self, obs, keep_gradients: bool) -> bool:
        import torch

        dist = torch.distributed.is_available() and torch.distributed.is_initialized()
        return (self.graph and not keep_gradients and not (dist and self.collective) and obs.is_cuda
                and all(hasattr(n, "predict_update_device") for n in self.nets))

    def _graph_key(self, obs, c0):
        params = tuple(p.data_ptr() for n in self.nets for p in n.parameters())
        return (tuple(obs.shape), tuple(c0.shape), params, id(self.engine))

    def _replay(self, obs, c0, key=None, clone: bool = True):
        import torch

        if key is None:
            key = self._graph_key(obs, c0)
        if self._g is not None and self._g[7] != self.engine.ws_generation:
            self._g = None  # the engine's workspace moved: the captured addresses are stale
        if self._g is None or self._g[0] != key:
            self._g = None
            if self.rho is not None and not isinstance(self.rho, torch.Tensor):
                self.rho = torch.as_tensor(np.asarray(self.rho, dtype=np.float64), device=obs.device)
            s_obs = obs.to(torch.float64).clone()
            s_c0 = c0.to(torch.float64).clone()
            side = torch.cuda.Stream(device=obs.device)
            side.wait_stream(torch.cuda.current_stream(obs.device))
            with torch.cuda.stream(side):  # warm-up: workspaces, cuDNN plans, kernel attributes
                for _ in range(2):
                    self._stages(s_obs, s_c0, False, False)
            torch.cuda.current_stream(obs.device).wait_stream(side)
            graph = torch.cuda.CUDAGraph()
            from . import _lib

            n0 = self.engine.launch_count + _lib.GLUE_LAUNCHES[0]
            with torch.cuda.graph(graph):
                maps, _, flags, cmax = self._stages(s_obs, s_c0, False, False)
            self._g = (key, graph, s_obs, s_c0, maps, (flags, cmax),
                       self.engine.launch_count + _lib.GLUE_LAUNCHES[0] - n0,
                       self.engine.ws_generation)
        _, graph, s_obs, s_c0, maps, (flags, cmax), n_launch, _ = self._g
        s_obs.copy_(obs)
        s_c0.copy_(c0)
        graph.replay()
        self.replayed_launches += n_launch  # the library's kernels inside the graph
        if not clone:  # the caller consumes the graph's own buffers before the next replay
            return maps, flags, cmax
        return [m.clone() for m in maps], flags.clone(), None if cmax is None else cmax.clone()

    def reconstruct(self, obs, c0, keep_gradients: bool = False, check_finite: bool = True):
        graphable = self._graphable(obs, keep_gradients)
        key = self._graph_key(obs, c0) if graphable else None
        if graphable and (self._g is not None and self._g[0] == key or self._seen == key):
            maps, flags, cmax = self._replay(obs, c0, key)
            grads = []
        else:
            self._seen = key
            maps, grads, flags, cmax = self._stages(obs, c0, keep_gradients, check_finite)
        if check_finite:
            self._check_stages(flags, cmax)  # first failing stage raises
        return (maps, grads) if keep_gradients else maps

    def reconstruct_host(self, obs, c0) -> np.ndarray:
        """:meth:`reconstruct` for the public API: the stage maps as one host array
        (K, B, nx, nz) f64.  The maps, the non-finite flags and the CFL maxima are
        copied to pinned host memory behind the stages on the stream, so the call
        has ONE device round trip; the checks run on the host copies."""
        import torch

        graphable = self._graphable(obs, False)
        key = self._graph_key(obs, c0) if graphable else None
        if graphable and (self._g is not None and self._g[0] == key or self._seen == key):
            maps, flags, cmax = self._replay(obs, c0, key, clone=False)
        else:
            self._seen = key
            maps, _, flags, cmax = self._stages(obs, c0, False, True)
        dev = torch.stack(maps)
        stage = _pinned(tuple(dev.shape), dev.device)
        stage.copy_(dev, non_blocking=True)
        small = flags.to(torch.float64).reshape(-1)
        n_flags = small.numel()
        if cmax is not None:
            small = torch.cat([small, cmax.to(torch.float64).reshape(-1)])
        small_host = _pinned((small.numel(),), dev.device)
        small_host.copy_(small, non_blocking=True)
        torch.cuda.current_stream(dev.device).synchronize()
        host_flags = small_host[:n_flags].to(flags.dtype).reshape(flags.shape)
        self._check_stages(host_flags, None if cmax is None else small_host[n_flags:].clone())
        return stage.numpy().copy()


_RECON_CACHE: dict = {}
_PINNED: dict = {}
_STAGE_EVENTS: dict = {}  # id(staging buffer) -> event after its last upload DMA


def _pinned(shape, device) -> "torch.Tensor":
    """Page-locked f64 host buffer of ``shape``, reused across calls (staging of
    the public API's host arrays: one memcpy in, one DMA to the device)."""
    import torch

    key = (tuple(shape), str(device))
    buf = _PINNED.get(key)
    if buf is None:
        if len(_PINNED) >= 8:
            _PINNED.pop(next(iter(_PINNED)))
        buf = _PINNED[key] = torch.empty(shape, dtype=torch.float64, pin_memory=True)
    return buf


def _upload(arrays, device) -> "torch.Tensor":
    """Host f64 arrays (stacked along axis 0) -> one device tensor through a
    pinned staging buffer.  Read-only ChannelData arrays are copied, never aliased."""
    import torch

    import warnings

    arrays = [np.asarray(a) for a in arrays]
    n = sum(a.shape[0] for a in arrays)
    stage = _pinned((n,) + arrays[0].shape[1:], device)
    ev = _STAGE_EVENTS.pop(id(stage), None)
    if ev is not None:
        ev.synchronize()  # the previous upload's DMA out of this buffer is done
    o = 0
    for a in arrays:
        with warnings.catch_warnings():  # read-only ChannelData arrays: only read here
            warnings.simplefilter("ignore", UserWarning)
            src = torch.from_numpy(a) if a.dtype == np.float64 else torch.from_numpy(a.astype(np.float64))
        stage[o:o + a.shape[0]].copy_(src)  # torch's multi-threaded host copy
        o += a.shape[0]
    # (uploading in pieces, each DMA behind the next piece's host copy, measured slower:
    # 0.31 against 0.16 ms for config 1's 4 MB of traces; small host copies are single-threaded)
    out = torch.empty(stage.shape, dtype=torch.float64, device=device)
    out.copy_(stage, non_blocking=True)
    # the staging buffer is reused by a later call: its next host write waits on this event
    ev = torch.cuda.Event()
    ev.record(torch.cuda.current_stream(device))
    _STAGE_EVENTS[id(stage)] = ev
    return out


def _download(maps) -> np.ndarray:
    """Stage maps (K tensors (B, nx, nz) on device) -> host (K, B, nx, nz) f64."""
    import torch

    dev = torch.stack(maps)
    stage = _pinned(tuple(dev.shape), dev.device)
    stage.copy_(dev, non_blocking=True)
    torch.cuda.current_stream(dev.device).synchronize()
    return stage.numpy().copy()


def _reconstructor(eng, nets, bounds, rho, collective: bool, grid) -> Reconstructor:
    """Reconstructor (and its captured graph) reused across calls with the same
    engine, networks and bounds; models with a density map are not cached."""
    if rho is not None:
        return Reconstructor(eng, nets, bounds, rho=rho, collective=collective, cfl_grid=grid)
    key = (id(eng), tuple(id(n) for n in nets), tuple(bounds), collective)
    rec = _RECON_CACHE.get(key)
    if rec is None or rec.engine is not eng or any(a is not b for a, b in zip(rec.nets, nets)):
        while len(_RECON_CACHE) >= 4:
            _RECON_CACHE.pop(next(iter(_RECON_CACHE)))
        rec = _RECON_CACHE[key] = Reconstructor(eng, nets, bounds, collective=collective,
                                                cfl_grid=grid)
    return rec


def unfold_infer(m_obs: ChannelData, c0: SosMap, nets, setup: InversionSetup) -> list[SosMap]:
    """Run all stages; returns C_1..C_K (unfold.py:253-267)."""
    import torch

    grid = c0.grid
    lo, hi = setup.bounds
    if not lo < hi:
        raise ValueError("bounds must satisfy c_min < c_max")
    damping = setup.damping if setup.damping is not None else zero_damping(grid)
    geometry = m_obs.geometry
    c_first = clamp_sos(c0, setup.bounds)
    # stage 1's input; later stages' inputs are checked on the device when the
    # clamp's upper bound lies above the CFL limit (Reconstructor.cfl_grid)
    _check_simulation_inputs(c_first, geometry, setup.pulse, damping)
    rho = None if setup.density is None else np.asarray(setup.density, dtype=np.float64)[None]
    eng = get_engine(grid, geometry.tx_nodes(), geometry.rx_nodes(), geometry.element_nodes,
                     setup.pulse.samples, damping, has_rho=rho is not None)
    # a per-sample call: never a hidden collective under torch.distributed
    rec = _reconstructor(eng, nets, setup.bounds, rho, collective=False, grid=grid)
    # ChannelData arrays are read-only views: a writable host copy for torch
    obs = _upload([m_obs.traces], eng.device)
    c = _upload([np.asarray(c0.values, dtype=np.float64)[None]], eng.device)
    try:
        host = rec.reconstruct_host(obs, c)
    except FloatingPointError as exc:
        raise NumericError(str(exc)) from exc
    return SosMap.stack_checked(grid, host[:, 0])


def unfold_infer_batch(m_obs_list, c0_list, nets, setup: InversionSetup) -> list[list[SosMap]]:
    """Batched extension of :func:`unfold_infer`: B phantoms on one acquisition,
    one launch set per stage for all of them.  Returns, per phantom, C_1..C_K.

    Under torch.distributed it is a collective: every rank passes the same lists,
    the (phantom, shot) units are sharded across ranks and the per-stage partial
    gradients combined with one all_reduce; every rank returns
    all maps.
    """
    import torch

    if len(m_obs_list) != len(c0_list) or not c0_list:
        raise ValueError("need one initial map per observed data set")
    grid = c0_list[0].grid
    lo, hi = setup.bounds
    if not lo < hi:
        raise ValueError("bounds must satisfy c_min < c_max")
    damping = setup.damping if setup.damping is not None else zero_damping(grid)
    geometry = m_obs_list[0].geometry
    for m, c0 in zip(m_obs_list, c0_list):
        if not m.geometry.same_acquisition(geometry):
            raise ValueError("batched inference needs one acquisition geometry")
        _check_simulation_inputs(clamp_sos(c0, setup.bounds), geometry, setup.pulse, damping)
    B = len(c0_list)
    rho = None if setup.density is None else np.broadcast_to(
        np.asarray(setup.density, dtype=np.float64), (B,) + grid.shape).copy()
    eng = get_engine(grid, geometry.tx_nodes(), geometry.rx_nodes(), geometry.element_nodes,
                     setup.pulse.samples, damping, n_phantoms=B, has_rho=rho is not None)
    rec = _reconstructor(eng, nets, setup.bounds, rho, collective=True, grid=grid)
    obs = _upload([m.traces for m in m_obs_list], eng.device)
    c = _upload([np.asarray(c0.values, np.float64)[None] for c0 in c0_list], eng.device)
    try:
        host = rec.reconstruct_host(obs, c)  # (K, B, nx, nz)
    except FloatingPointError as exc:
        raise NumericError(str(exc)) from exc
    return [SosMap.stack_checked(grid, host[:, b]) for b in range(B)]
