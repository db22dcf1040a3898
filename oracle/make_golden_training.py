"""Golden fixtures for the training-side rows, made by
running the REAL reference package.

TEST INFRASTRUCTURE, run in the build container (the reference is absent on
GPU boxes):

    python oracle/make_golden_training.py

Writes tests/golden/training.npz and tests/golden/raster_*.fwir:
* FWIR rasters written by ``fwilab.raster.write_raster`` (f32, f64, u8, rank 0-4)
  — the byte-level format our reader/writer must reproduce;
* one ``fwilab.network.train_step`` on a 10x12 batch of two samples for
  ``UpdateNetwork.initialize(seed=7)``: the loss, per-layer sums / sampled
  entries of the parameter gradients (from the reference's own
  _forward_pass/_backward_pass, exactly as train_step accumulates them) and of
  the parameters after the Adam step, plus hashes of the initial parameters
  (so RefUpdateNet.initialize is checked bit for bit);
* the reference's block-dataset round trip: BlockDataset.save bytes.
"""

from __future__ import annotations

import hashlib
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
REF_SRC = "/root/reference/pkg/src"
OUT = ROOT / "tests" / "golden"
SAMPLE = 64  # sampled entries per parameter tensor


def main() -> None:
    sys.path.insert(0, REF_SRC)
    from fwilab import network as nw
    from fwilab import raster as rs
    from fwilab.unfold import BlockDataset

    OUT.mkdir(parents=True, exist_ok=True)
    rng = np.random.default_rng(2024)
    # ---- FWIR rasters
    arrays = {
        "f32_r2": rng.standard_normal((3, 5)).astype(np.float32),
        "f64_r3": rng.standard_normal((2, 3, 4)),
        "u8_r1": rng.integers(0, 255, size=7).astype(np.uint8),
        "f64_r0": np.array(3.25),
        "f32_r4": rng.standard_normal((2, 1, 3, 2)).astype(np.float32),
    }
    for name, a in arrays.items():
        rs.write_raster(OUT / f"raster_{name}.fwir", a)

    # ---- one train_step of the reference network
    nx, nz, n = 10, 12, 2
    net = nw.UpdateNetwork.initialize(seed=7)
    init_hash = [hashlib.sha256(p.tobytes()).hexdigest() for p in net.parameters()]
    batch = []
    for _ in range(n):
        c = 1500.0 + 40.0 * rng.standard_normal((nx, nz))
        g = 1e-3 * rng.standard_normal((nx, nz))
        gt = 1500.0 + 60.0 * rng.standard_normal((nx, nz))
        batch.append((c, g, gt))
    # gradients exactly as train_step accumulates them (network.py:268-346)
    dtype = net.dtype
    grad_sum = None
    total = 0.0
    for c_k, g_k, c_gt in batch:
        x = np.stack([nw.normalize_sos(c_k, net.norm).astype(dtype),
                      nw.normalize_gradient(g_k).astype(dtype)])
        h, caches = nw._forward_pass(net, x, want_cache=True)
        err = c_gt - (c_k + h.astype(np.float64) * net.norm.scale)
        total += float(np.sum(err * err))
        dh = (-2.0 * net.norm.scale / n) * err
        _, grads = nw._backward_pass(net, dh.astype(dtype), caches)
        grad_sum = grads if grad_sum is None else [a + b for a, b in zip(grad_sum, grads)]
    lr = 1e-3
    after = net.copy()
    adam = nw.AdamState.for_network(after)
    loss = nw.train_step(after, batch, adam, lr)
    assert abs(loss - total / n) <= 1e-12 * abs(loss)
    pick = [np.sort(np.random.default_rng(i).choice(p.size, size=min(SAMPLE, p.size), replace=False))
            for i, p in enumerate(net.parameters())]
    out = {
        "nx": nx, "nz": nz, "seed": 7, "lr": lr, "loss": loss,
        "c": np.stack([b[0] for b in batch]), "g": np.stack([b[1] for b in batch]),
        "gt": np.stack([b[2] for b in batch]),
        "init_sha256": np.array(init_hash),
        "grad_sums": np.array([float(np.sum(gr.astype(np.float64))) for gr in grad_sum]),
        "grad_norms": np.array([float(np.linalg.norm(gr.astype(np.float64))) for gr in grad_sum]),
    }
    for i, (gr, p_after, idx) in enumerate(zip(grad_sum, after.parameters(), pick)):
        out[f"idx_{i}"] = idx
        out[f"grad_{i}"] = gr.reshape(-1)[idx]
        out[f"after_{i}"] = p_after.reshape(-1)[idx]
    # the reference Adam step applied to its own gradients, for a bit-exact optimizer check
    np.savez_compressed(OUT / "training.npz", **out)

    # ---- block dataset bytes
    ds = BlockDataset(2, rng.standard_normal((2, 3, 4)), rng.standard_normal((2, 3, 4)),
                      rng.standard_normal((2, 3, 4)))
    ds.save(OUT / "block_stage")
    print("wrote", sorted(p.name for p in OUT.glob("raster_*.fwir")), "training.npz, block_stage/")


if __name__ == "__main__":
    main()
