"""Learned update of the unfolded iteration — kept in PyTorch, as the north star asks.

The reference's update network is a NumPy CNN (network.py:1-15).  Only its
interface is on the hot path: ``predict_update(c_values, g_values)`` with the
normalisation ``(c - offset)/scale``, ``g / max|g|`` and ``h * scale``
(network.py:43-68, 224-229).  :class:`UpdateCNN` implements that interface
for the config-1 architecture (4 layers of 3x3 convolutions, 32 channels,
inputs (C, g)), and additionally ``predict_update_device`` so the unfolded
loop never leaves the GPU.  TF32 is disabled for its convolutions so the fp32
network is an fp32 computation.
"""

from __future__ import annotations

import os
from dataclasses import dataclass

import numpy as np
import torch
from torch import nn

__all__ = ["NormSpec", "normalize_sos", "normalize_gradient", "denormalize_update", "UpdateCNN",
           "make_update_nets"]


@dataclass(frozen=True)
class NormSpec:
    """Speed offset/scale of the network input and output (network.py:43-53)."""

    offset: float = 1400.0
    scale: float = 666.0

    def __post_init__(self):
        if not self.scale > 0:
            raise ValueError("scale must be positive")


def normalize_sos(c: np.ndarray, spec: NormSpec) -> np.ndarray:
    return (np.asarray(c, dtype=np.float64) - spec.offset) / spec.scale


def normalize_gradient(g: np.ndarray) -> np.ndarray:
    """Unit max-magnitude gradient, zeros stay zeros (network.py:60-64)."""
    g = np.asarray(g, dtype=np.float64)
    peak = np.abs(g).max()
    return g / peak if peak > 0 else np.zeros_like(g)


def denormalize_update(h: np.ndarray, spec: NormSpec) -> np.ndarray:
    return np.asarray(h, dtype=np.float64) * spec.scale


class UpdateCNN(nn.Module):
    """Conv(2,ch,3)-ReLU-[Conv(ch,ch,3)-ReLU]x(layers-2)-Conv(ch,1,3), zero padding."""

    def __init__(self, channels: int = 32, layers: int = 4, norm: NormSpec | None = None):
        super().__init__()
        if layers < 2:
            raise ValueError("need at least two layers")
        mods: list[nn.Module] = [nn.Conv2d(2, channels, 3, padding=1), nn.ReLU()]
        for _ in range(layers - 2):
            mods += [nn.Conv2d(channels, channels, 3, padding=1), nn.ReLU()]
        mods.append(nn.Conv2d(channels, 1, 3, padding=1))
        self.body = nn.Sequential(*mods)
        self.norm = norm or NormSpec()

    # cuDNN's fused convolution + bias + ReLU for the hidden layers on the device
    # (one launch per layer instead of three); DUFWI_FUSED_CONV=0 runs the modules
    fused_conv = os.environ.get("DUFWI_FUSED_CONV", "1") != "0"

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        with torch.backends.cudnn.flags(enabled=True, allow_tf32=False):
            # (inference only: the fused op has no backward)
            if not (self.fused_conv and x.is_cuda and x.dtype == torch.float32
                    and not torch.is_grad_enabled()):
                return self.body(x)
            mods = list(self.body)
            for k, m in enumerate(mods):
                if isinstance(m, nn.Conv2d):
                    if k + 1 < len(mods) and isinstance(mods[k + 1], nn.ReLU):
                        x = torch.cudnn_convolution_relu(x.contiguous(), m.weight, m.bias, m.stride,
                                                         m.padding, m.dilation, m.groups)
                    else:
                        x = m(x)
            return x

    @torch.no_grad()
    def predict_update_device(self, c: torch.Tensor, g: torch.Tensor) -> torch.Tensor:
        """Update in m/s for maps (..., nx, nz) on the module's device (f64 in, f64 out)."""
        squeeze = c.dim() == 2
        c4 = c.reshape(-1, 1, *c.shape[-2:])
        g4 = g.reshape(-1, 1, *g.shape[-2:])
        peak = g4.abs().amax(dim=(1, 2, 3), keepdim=True)
        gn = torch.where(peak > 0, g4 / torch.where(peak > 0, peak, torch.ones_like(peak)),
                         torch.zeros_like(g4))
        cn = (c4 - self.norm.offset) / self.norm.scale
        dtype = next(self.parameters()).dtype
        h = self(torch.cat([cn, gn], dim=1).to(dtype)).to(torch.float64) * self.norm.scale
        return h.reshape(c.shape[-2:]) if squeeze else h.reshape(c.shape)

    @torch.no_grad()
    def stage_device(self, c: torch.Tensor, g: torch.Tensor, lo: float, hi: float) -> torch.Tensor:
        """One unfolded stage on the device: clamp(c + predict_update_device(c, g), lo, hi)
        (unfold.py:263-265), with the input normalisation and the update in libdufwi:
        three launches instead of ~15 elementwise ones, the same f64 operations (bits)."""
        from . import _lib

        if next(self.parameters()).dtype != torch.float32 or not c.is_cuda:
            return torch.clamp(c + self.predict_update_device(c, g), lo, hi)
        so = _lib.lib()
        c = c.to(torch.float64).contiguous()
        g = g.to(torch.float64).contiguous()
        nx, nz = c.shape[-2:]
        n = nx * nz
        B = c.numel() // n
        x = torch.empty((B, 2, nx, nz), dtype=torch.float32, device=c.device)
        peak = torch.empty(B, dtype=torch.float64, device=c.device)
        stream = torch.cuda.current_stream(c.device).cuda_stream
        _lib.check(so.dufwi_net_input(c.data_ptr(), g.data_ptr(), B, n, float(self.norm.offset),
                                      float(self.norm.scale), peak.data_ptr(), x.data_ptr(), stream))
        h = self(x).contiguous()
        out = torch.empty_like(c)
        _lib.check(so.dufwi_apply_update(c.data_ptr(), h.data_ptr(), c.numel(),
                                         float(self.norm.scale), float(lo), float(hi),
                                         out.data_ptr(), stream))
        _lib.GLUE_LAUNCHES[0] += 3
        return out

    def predict_update(self, c_values: np.ndarray, g_values: np.ndarray) -> np.ndarray:
        """Reference interface (network.py:224-229): numpy in, numpy out."""
        dev = next(self.parameters()).device
        c = torch.as_tensor(np.asarray(c_values, dtype=np.float64), device=dev)
        g = torch.as_tensor(np.asarray(g_values, dtype=np.float64), device=dev)
        return self.predict_update_device(c, g).cpu().numpy()


def make_update_nets(k: int, seed: int = 0, channels: int = 32, layers: int = 4,
                     device=None, dtype=torch.float32) -> list[UpdateCNN]:
    """K random-init stage networks, stage j seeded with ``torch.manual_seed(seed + j)``."""
    nets = []
    for j in range(k):
        torch.manual_seed(seed + j)
        net = UpdateCNN(channels, layers).to(dtype)
        if device is not None:
            net = net.to(device)
        nets.append(net.eval())
    return nets
