"""Training side of DUFWI on the GPU physics step.

Block-wise training never backpropagates through the wave solver: for every
training sample the current estimate and its misfit gradient are materialised
first, then the stage network is fit as a supervised regression onto the
ground truth (reference unfold.py:1-10).  The physics part — one gradient
evaluation per sample and stage — is the dominant training cost
(PAPER.md:201), so here it runs batched: all samples of a stage share one
acquisition, so B samples are B phantoms of ONE engine launch set (one
forward + adjoint sweep over B x S units) instead of B sequential
``compute_gradient`` calls.  The learned update and the regression step stay
in PyTorch.

Mirrors, with the reference's names, signatures and failure semantics:

* ``UnfoldPlan``, ``BlockDataset`` (save/load as FWIR rasters)  — unfold.py:46-115
* ``_roll_estimate``, ``prepare_block_dataset``, ``advance_block_dataset``
  (a sample whose physics pass fails is skipped with a log entry)  — unfold.py:145-213
* ``train_step`` (mean per-sample squared reconstruction error, gradients
  through the output rescaling, Adam with float64 moments)  — network.py:268-346
* ``train_block``, ``train_all_blocks``  — unfold.py:216-300
* ``simulate_dataset``: the forward-only sweeps of dataset generation
  (datagen.py:184-204 calls simulate_all once per sample), batched over
  samples, channel data written as FWIR  — SURVEY §8(f) row 2.

``RefUpdateNet`` is a PyTorch restatement of the reference's six-layer 5x5
CNN (network.py:1-15, 155-200) with its seeded initialisation, so a
reference-trained network can be imported and trained further here.
"""

from __future__ import annotations

import logging
import os
from dataclasses import dataclass
from pathlib import Path

import numpy as np
import torch
from torch import nn

from .forward import DampingProfile, _check_simulation_inputs, get_engine, zero_damping
from .grid import ChannelData, SosMap, check_cfl, homogeneous_map
from .network import NormSpec
from .raster import read_raster, write_raster
from .unfold import InversionSetup, clamp_sos

logger = logging.getLogger(__name__)

__all__ = ["UnfoldPlan", "BlockDataset", "DEFAULT_LR_SCHEDULE", "batched_gradients",
           "prepare_block_dataset", "advance_block_dataset", "train_step", "AdamState",
           "train_block", "train_all_blocks", "RefUpdateNet", "simulate_dataset"]

#: Default learning-rate schedule for the five-stage configuration (unfold.py:43).
DEFAULT_LR_SCHEDULE = (1e-4, 1e-4, 5e-5, 1e-5, 1e-5)


@dataclass(frozen=True)
class UnfoldPlan:
    """Stage count, per-stage learning rates, per-block epoch budget (unfold.py:46-63)."""

    k: int = 5
    lr_schedule: tuple[float, ...] = DEFAULT_LR_SCHEDULE
    epochs: int = 40
    batch_size: int = 32

    def __post_init__(self):
        if self.k < 1:
            raise ValueError("need at least one stage")
        if len(self.lr_schedule) != self.k:
            raise ValueError(f"lr_schedule has {len(self.lr_schedule)} entries for k={self.k}")
        if self.epochs < 1 or self.batch_size < 1:
            raise ValueError("epochs and batch_size must be >= 1")


@dataclass
class BlockDataset:
    """Aligned (C_k, g_k, C_gt) stacks for one training stage (unfold.py:76-115)."""

    k: int
    c_maps: np.ndarray     # (N, nx, nz)
    gradients: np.ndarray  # (N, nx, nz)
    targets: np.ndarray    # (N, nx, nz)

    def __post_init__(self):
        if not (self.c_maps.shape == self.gradients.shape == self.targets.shape):
            raise ValueError("dataset stacks must share one shape")
        if self.c_maps.ndim != 3:
            raise ValueError("dataset stacks must be (N, nx, nz)")

    def __len__(self) -> int:
        return self.c_maps.shape[0]

    def sample(self, i: int):
        return self.c_maps[i], self.gradients[i], self.targets[i]

    def save(self, directory) -> None:
        d = Path(directory)
        d.mkdir(parents=True, exist_ok=True)
        write_raster(d / "c_maps.fwir", self.c_maps)
        write_raster(d / "gradients.fwir", self.gradients)
        write_raster(d / "targets.fwir", self.targets)
        write_raster(d / "stage.fwir", np.array([self.k], dtype=np.float64))

    @classmethod
    def load(cls, directory) -> "BlockDataset":
        d = Path(directory)
        return cls(k=int(read_raster(d / "stage.fwir")[0]),
                   c_maps=read_raster(d / "c_maps.fwir"),
                   gradients=read_raster(d / "gradients.fwir"),
                   targets=read_raster(d / "targets.fwir"))


# ------------------------------------------------------------------ physics
def _engine_for(samples, setup: InversionSetup, n_phantoms: int):
    m_obs = samples[0][0]
    geometry = m_obs.geometry
    grid = geometry.grid
    damping = setup.damping if setup.damping is not None else zero_damping(grid)
    eng = get_engine(grid, geometry.tx_nodes(), geometry.rx_nodes(), geometry.element_nodes,
                     setup.pulse.samples, damping, n_phantoms=n_phantoms,
                     has_rho=getattr(setup, "density", None) is not None)
    return eng, damping


def _sample_ok(c: np.ndarray, m_obs: ChannelData, setup: InversionSetup, damping) -> str | None:
    """The reference's per-sample input checks (forward.py:256-270); message or None."""
    try:
        _check_simulation_inputs(SosMap(m_obs.geometry.grid, c), m_obs.geometry, setup.pulse,
                                 damping)
    except ValueError as exc:
        return str(exc)
    return None


def batched_gradients(c_maps, samples, setup: InversionSetup, batch: int | None = None):
    """Misfit gradients of ``compute_gradient(C_i, m_obs_i, pulse, damping)`` for all i.

    ``c_maps`` (N, nx, nz); ``samples`` the matching (m_obs, c_gt) pairs, all on
    one acquisition geometry.  Runs ``batch`` samples per engine launch set
    (default: all).  Returns (gradients (N, nx, nz) float64 numpy, ok (N,) bool):
    a sample is not ok when its inputs fail the reference's checks or its misfit
    or gradient is non-finite (what makes ``compute_gradient`` raise).
    """
    c_maps = np.asarray(c_maps, dtype=np.float64)
    n = c_maps.shape[0]
    if n != len(samples):
        raise ValueError("maps and samples are misaligned")
    geometry = samples[0][0].geometry
    for m_obs, _ in samples:
        if not m_obs.geometry.same_acquisition(geometry):
            raise ValueError("batched gradients need one acquisition geometry for all samples")
    batch = n if batch is None else max(1, int(batch))
    grads = np.zeros_like(c_maps)
    ok = np.ones(n, dtype=bool)
    rho = getattr(setup, "density", None)
    for a in range(0, n, batch):
        idx = list(range(a, min(n, a + batch)))
        eng, damping = _engine_for(samples, setup, len(idx))
        for i in idx:
            why = _sample_ok(c_maps[i], samples[i][0], setup, damping)
            if why is not None:
                ok[i] = False
                logger.warning("sample %d: %s", i, why)
        # failing samples still ride along (with a benign map) so the batch shape stays fixed
        c = np.stack([c_maps[i] if ok[i] else np.full(c_maps[i].shape, 1500.0) for i in idx])
        rho_b = None if rho is None else np.broadcast_to(np.asarray(rho, np.float64),
                                                         c.shape).copy()
        eng.set_model(c, rho_b)
        obs = torch.from_numpy(np.concatenate([np.require(samples[i][0].traces, np.float64,
                                                          ["C", "W"]) for i in idx]))
        misfit, g = eng.misfit_and_gradient(obs.to(eng.device), check_finite=False)
        fin = (torch.isfinite(g).flatten(1).all(dim=1) & torch.isfinite(misfit)).cpu().numpy()
        g_host = g.cpu().numpy()
        for j, i in enumerate(idx):
            if ok[i] and not fin[j]:
                ok[i] = False
                logger.warning("sample %d: non-finite misfit or gradient", i)
            if ok[i]:
                grads[i] = g_host[j]
    return grads, ok


def _predict(net, c: np.ndarray, g: np.ndarray) -> np.ndarray:
    """Stage update for a stack of maps: the reference interface predict_update(c, g)."""
    if hasattr(net, "predict_update_device"):
        dev = next(net.parameters()).device
        return net.predict_update_device(torch.as_tensor(c, device=dev),
                                         torch.as_tensor(g, device=dev)).cpu().numpy()
    return np.stack([net.predict_update(ci, gi) for ci, gi in zip(c, g)])


def _clamp(c: np.ndarray, bounds) -> np.ndarray:
    lo, hi = bounds
    if not lo < hi:
        raise ValueError("bounds must satisfy c_min < c_max")
    return np.clip(c, lo, hi)


def _roll_estimate(m_obs: ChannelData, nets, setup: InversionSetup, upto: int):
    """Run ``upto`` trained stages from the water map; returns (C_upto, gradient)
    (unfold.py:145-160).  Single-sample form of :func:`prepare_block_dataset`."""
    c, g, ok = _roll_batch([(m_obs, None)], nets, setup, upto)
    if not ok[0]:
        from .forward import NumericError
        raise NumericError("physics pass failed while rolling the estimate")
    return SosMap(m_obs.geometry.grid, c[0]), g[0]


def _roll_batch(samples, nets, setup: InversionSetup, upto: int, batch: int | None = None):
    grid = samples[0][0].geometry.grid
    c0 = clamp_sos(homogeneous_map(grid, setup.water_speed), setup.bounds).values
    c = np.broadcast_to(c0, (len(samples),) + grid.shape).copy()
    ok = np.ones(len(samples), dtype=bool)
    for j in range(upto):
        g, okj = batched_gradients(c, samples, setup, batch)
        ok &= okj
        c = _clamp(c + _predict(nets[j], c, g), setup.bounds)
    g, okj = batched_gradients(c, samples, setup, batch)
    return c, g, ok & okj


def prepare_block_dataset(k: int, samples, nets, setup: InversionSetup,
                          batch: int | None = None) -> BlockDataset:
    """Materialise stage-``k`` tuples by replaying stages 0..k-1 (unfold.py:163-187).

    Samples whose physics pass fails are skipped with a log entry."""
    if k < 0 or k > len(nets):
        raise ValueError(f"stage {k} requires {k} trained networks, have {len(nets)}")
    c, g, ok = _roll_batch(samples, nets, setup, k, batch)
    for i in np.flatnonzero(~ok):
        logger.error("sample %d skipped while preparing stage %d", i, k)
    if not ok.any():
        raise RuntimeError(f"no usable samples while preparing stage {k}")
    targets = np.stack([np.asarray(s[1].values, np.float64) for s in samples])
    return BlockDataset(k, c[ok], g[ok], targets[ok])


def advance_block_dataset(ds: BlockDataset, net, samples, setup: InversionSetup,
                          batch: int | None = None) -> BlockDataset:
    """Roll a stage dataset forward through one trained network: one batched
    gradient pass over all samples (unfold.py:190-213)."""
    if len(ds) != len(samples):
        raise ValueError("dataset and sample list are misaligned")
    grid = samples[0][0].geometry.grid
    c = _clamp(ds.c_maps + _predict(net, ds.c_maps, ds.gradients), setup.bounds)
    for ci in c:
        SosMap(grid, ci)  # the reference's SosMap validation (grid.py:94-105)
    g, ok = batched_gradients(c, samples, setup, batch)
    if not ok.all():
        from .forward import NumericError
        raise NumericError(f"physics pass failed for samples {np.flatnonzero(~ok).tolist()}")
    return BlockDataset(ds.k + 1, c, g, ds.targets.copy())


# ---------------------------------------------------------------- training
class AdamState:
    """Adam with float64 moments and the reference's update (network.py:240-266):
    p -= lr * (m / (1 - b1^t)) / (sqrt(v / (1 - b2^t)) + eps), cast to p's dtype."""

    def __init__(self, params, beta1=0.9, beta2=0.999, eps=1e-8):
        self.params = list(params)
        self.m = [torch.zeros_like(p, dtype=torch.float64) for p in self.params]
        self.v = [torch.zeros_like(p, dtype=torch.float64) for p in self.params]
        self.t = 0
        self.beta1, self.beta2, self.eps = beta1, beta2, eps

    @torch.no_grad()
    def step(self, grads, lr: float) -> None:
        if len(grads) != len(self.params):
            raise ValueError("parameter/gradient count mismatch")
        self.t += 1
        bc1 = 1.0 - self.beta1 ** self.t
        bc2 = 1.0 - self.beta2 ** self.t
        for p, g, m, v in zip(self.params, grads, self.m, self.v):
            g64 = g.to(torch.float64)
            m.mul_(self.beta1).add_((1.0 - self.beta1) * g64)
            v.mul_(self.beta2).add_((1.0 - self.beta2) * g64 * g64)
            p.sub_((lr * (m / bc1) / (torch.sqrt(v / bc2) + self.eps)).to(p.dtype))


def _normalized_inputs(c_k: torch.Tensor, g_k: torch.Tensor, norm: NormSpec, dtype):
    cn = (c_k - norm.offset) / norm.scale
    peak = g_k.abs().flatten(1).amax(dim=1).view(-1, 1, 1)
    gn = torch.where(peak > 0, g_k / torch.where(peak > 0, peak, torch.ones_like(peak)),
                     torch.zeros_like(g_k))
    return torch.stack([cn, gn], dim=1).to(dtype)


def train_step(net: nn.Module, batch, adam: AdamState, lr: float) -> float:
    """One Adam step on the mean per-sample squared reconstruction error
    (network.py:268-346): loss_i = sum((C_gt - (C_k + scale * H))^2), gradients
    through the output rescaling.  ``batch``: (C_k, g_k, C_gt) triples (numpy or
    tensors, m/s).  Returns the batch loss before the step."""
    if not len(batch):
        raise ValueError("batch must not be empty")
    p0 = next(net.parameters())
    dev, dtype = p0.device, p0.dtype
    ck = torch.stack([torch.as_tensor(np.asarray(b[0]), dtype=torch.float64) for b in batch]).to(dev)
    gk = torch.stack([torch.as_tensor(np.asarray(b[1]), dtype=torch.float64) for b in batch]).to(dev)
    gt = torch.stack([torch.as_tensor(np.asarray(b[2]), dtype=torch.float64) for b in batch]).to(dev)
    if not (ck.shape == gk.shape == gt.shape):
        raise ValueError("inconsistent sample shapes")
    norm = getattr(net, "norm", NormSpec())
    x = _normalized_inputs(ck, gk, norm, dtype)
    params = [p for p in net.parameters()]
    for p in params:
        p.grad = None
    with torch.backends.cudnn.flags(enabled=True, allow_tf32=False):
        h = net(x)[:, 0].to(torch.float64)
    err = gt - (ck + h * norm.scale)
    per = (err * err).flatten(1).sum(dim=1)
    loss = per.mean()
    if not bool(torch.isfinite(per).all()):
        bad = int(torch.nonzero(~torch.isfinite(per))[0, 0])
        raise FloatingPointError(f"non-finite loss at batch sample {bad}")
    loss.backward()
    adam.step([p.grad for p in params], lr)
    return float(loss.item())


def train_block(k: int, ds: BlockDataset, plan: UnfoldPlan, seed: int, net_factory=None,
                device=None):
    """Fit stage ``k``'s network on its dataset: final-epoch network and per-epoch mean
    losses (unfold.py:216-250); shuffling from SeedSequence([seed, k]) as the reference."""
    if len(ds) == 0:
        raise ValueError("empty block dataset")
    init_seed, shuffle_seed = np.random.SeedSequence([seed, k]).spawn(2)
    s0 = int(init_seed.generate_state(1)[0])
    if net_factory is None:
        net = RefUpdateNet.initialize(s0)
    else:
        net = net_factory(s0)
    if device is not None:
        net = net.to(device)
    adam = AdamState(net.parameters())
    rng = np.random.default_rng(shuffle_seed)
    lr = plan.lr_schedule[k]
    losses_epoch = []
    n = len(ds)
    for epoch in range(plan.epochs):
        order = rng.permutation(n)
        losses = []
        for start in range(0, n, plan.batch_size):
            idx = order[start:start + plan.batch_size]
            try:
                losses.append(train_step(net, [ds.sample(int(i)) for i in idx], adam, lr))
            except FloatingPointError as exc:
                raise FloatingPointError(
                    f"stage {k} diverged at epoch {epoch}, batch {start // plan.batch_size}") from exc
        losses_epoch.append(float(np.mean(losses)))
    return net, losses_epoch


def train_all_blocks(samples, plan: UnfoldPlan, setup: InversionSetup, seed: int,
                     dataset_dir=None, net_factory=None, device=None, batch: int | None = None):
    """Train all stages in sequence, advancing the materialised dataset through each
    freshly trained network (unfold.py:268-300); ``dataset_dir`` keeps each stage."""
    nets, histories = [], []
    ds = prepare_block_dataset(0, samples, nets, setup, batch)
    for k in range(plan.k):
        if dataset_dir is not None:
            ds.save(Path(dataset_dir) / f"stage_{k:02d}")
        net, losses = train_block(k, ds, plan, seed, net_factory, device)
        nets.append(net)
        histories.append(losses)
        logger.info("stage %d trained: first %.4g last %.4g", k, losses[0], losses[-1])
        if k + 1 < plan.k:
            ds = advance_block_dataset(ds, net, samples, setup, batch)
    return nets, histories


# ------------------------------------------------- reference network in torch
class RefUpdateNet(nn.Module):
    """The reference's update network (network.py:1-15): conv 5x5 2->64->128->256
    with ReLU, the three maps concatenated (448) -> 128 -> 64 (ReLU) -> 1 (linear),
    zero padding.  ``initialize(seed)`` reproduces UpdateNetwork.initialize
    (fan-in uniform weights from default_rng(seed), zero biases)."""

    STAGE1 = (64, 128, 256)
    STAGE2 = (128, 64, 1)

    def __init__(self, norm: NormSpec | None = None, dtype=torch.float32):
        super().__init__()
        s1, s2 = self.STAGE1, self.STAGE2
        plan = [(2, s1[0]), (s1[0], s1[1]), (s1[1], s1[2]), (sum(s1), s2[0]), (s2[0], s2[1]),
                (s2[1], s2[2])]
        self.convs = nn.ModuleList(nn.Conv2d(i, o, 5, padding=2, dtype=dtype) for i, o in plan)
        self.norm = norm or NormSpec()

    @staticmethod
    def layer_plan():
        s1, s2 = RefUpdateNet.STAGE1, RefUpdateNet.STAGE2
        return [(2, s1[0]), (s1[0], s1[1]), (s1[1], s1[2]), (sum(s1), s2[0]), (s2[0], s2[1]),
                (s2[1], s2[2])]

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        r = torch.relu
        a1 = r(self.convs[0](x))
        a2 = r(self.convs[1](a1))
        a3 = r(self.convs[2](a2))
        h = r(self.convs[3](torch.cat([a1, a2, a3], dim=1)))
        h = r(self.convs[4](h))
        return self.convs[5](h)

    @classmethod
    def from_arrays(cls, kernels, biases, norm: NormSpec | None = None, dtype=torch.float32):
        """Import (out, in, 5, 5) kernels and biases, e.g. a reference UpdateNetwork's."""
        net = cls(norm, dtype)
        with torch.no_grad():
            for conv, k, b in zip(net.convs, kernels, biases):
                conv.weight.copy_(torch.as_tensor(np.asarray(k)))
                conv.bias.copy_(torch.as_tensor(np.asarray(b)))
        return net

    @classmethod
    def initialize(cls, seed: int, norm: NormSpec | None = None, dtype=np.float32):
        rng = np.random.default_rng(seed)
        ks, bs = [], []
        for c_in, c_out in cls.layer_plan():
            bound = 1.0 / np.sqrt(c_in * 25)
            ks.append(rng.uniform(-bound, bound, size=(c_out, c_in, 5, 5)).astype(dtype))
            bs.append(np.zeros(c_out, dtype=dtype))
        return cls.from_arrays(ks, bs, norm, torch.float32 if dtype == np.float32 else torch.float64)

    @torch.no_grad()
    def predict_update_device(self, c: torch.Tensor, g: torch.Tensor) -> torch.Tensor:
        squeeze = c.dim() == 2
        c3 = c.reshape(-1, *c.shape[-2:]).to(torch.float64)
        g3 = g.reshape(-1, *g.shape[-2:]).to(torch.float64)
        dtype = next(self.parameters()).dtype
        with torch.backends.cudnn.flags(enabled=True, allow_tf32=False):
            h = self(_normalized_inputs(c3, g3, self.norm, dtype))[:, 0].to(torch.float64)
        h = h * self.norm.scale
        return h.reshape(c.shape[-2:]) if squeeze else h.reshape(c.shape)

    def predict_update(self, c_values: np.ndarray, g_values: np.ndarray) -> np.ndarray:
        dev = next(self.parameters()).device
        return self.predict_update_device(torch.as_tensor(np.asarray(c_values, np.float64), device=dev),
                                          torch.as_tensor(np.asarray(g_values, np.float64), device=dev)
                                          ).cpu().numpy()


# ------------------------------------------------------- dataset forwards
def simulate_dataset(sos_maps, geometry, pulse, damping: DampingProfile | None = None,
                     out_dir=None, batch: int | None = None, density=None):
    """Channel data of many ground-truth maps on one acquisition: the forward-only
    sweeps of dataset generation (datagen.py:184-204 runs simulate_all per sample),
    batched as phantoms of one engine launch set, no wavefield storage (16 B per
    cell update).  Returns the list of ChannelData; with ``out_dir`` also writes
    ``sample_{i:06d}/sos.fwir`` and ``cd.fwir`` as the reference's layout."""
    maps = [m if isinstance(m, SosMap) else SosMap(geometry.grid, m) for m in sos_maps]
    grid = geometry.grid
    damping = damping if damping is not None else zero_damping(grid)
    for m in maps:
        _check_simulation_inputs(m, geometry, pulse, damping)
    n = len(maps)
    batch = n if batch is None else max(1, int(batch))
    S = len(geometry.tx_nodes())
    out = []
    for a in range(0, n, batch):
        idx = list(range(a, min(n, a + batch)))
        eng = get_engine(grid, geometry.tx_nodes(), geometry.rx_nodes(), geometry.element_nodes,
                         pulse.samples, damping, n_phantoms=len(idx), has_rho=density is not None)
        rho = None
        if density is not None:
            rho = np.stack([np.asarray(density[i], np.float64) for i in idx])
        eng.set_model(np.stack([maps[i].values for i in idx]), rho)
        tr = eng.forward(units=(0, eng.n_units)).double().cpu().numpy()
        for j, i in enumerate(idx):
            cd = ChannelData(tr[j * S:(j + 1) * S], geometry, grid.dt)
            out.append(cd)
            if out_dir is not None:
                d = Path(out_dir) / f"sample_{i:06d}"
                d.mkdir(parents=True, exist_ok=True)
                write_raster(d / "sos.fwir", maps[i].values)
                write_raster(d / "cd.fwir", cd.traces)
    return out
