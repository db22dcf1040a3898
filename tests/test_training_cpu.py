"""Training-side rows on CPU, pinned to fixtures made
by running the reference (oracle/make_golden_training.py):

* FWIR rasters: our reader returns the reference's arrays and our writer its bytes;
* BlockDataset.save/load reproduces the reference's stage files byte for byte;
* RefUpdateNet.initialize(seed) equals UpdateNetwork.initialize(seed) bit for bit;
* train_step: loss and parameter gradients of the reference's train_step (torch
  fp32 convolutions vs numpy im2col sgemm: rounding-level tolerance), and the
  Adam update formula bit for bit on the reference's own gradient values.
"""

from __future__ import annotations

import hashlib
import io

import numpy as np
import pytest
import torch

from paper_2603_04070_b200 import raster
from paper_2603_04070_b200.training import (AdamState, BlockDataset, RefUpdateNet, UnfoldPlan,
                                            train_block, train_step)

from .conftest import GOLDEN

ARRAYS = ["f32_r2", "f64_r3", "u8_r1", "f64_r0", "f32_r4"]


@pytest.mark.parametrize("name", ARRAYS)
def test_raster_roundtrip_matches_reference_bytes(name):
    blob = (GOLDEN / f"raster_{name}.fwir").read_bytes()
    a = raster.read_raster(GOLDEN / f"raster_{name}.fwir")
    assert raster.encode_raster(a) == blob
    buf = io.BytesIO()
    raster.write_raster(buf, a)
    assert buf.getvalue() == blob
    b = raster.read_raster(io.BytesIO(blob))
    assert b.dtype == a.dtype and b.shape == a.shape and np.array_equal(a, b)


def test_raster_errors():
    good = (GOLDEN / "raster_f64_r3.fwir").read_bytes()
    with pytest.raises(raster.RasterFormatError, match="bad magic"):
        raster.decode_raster(b"XXXX" + good[4:])
    with pytest.raises(raster.RasterFormatError, match="truncated header"):
        raster.decode_raster(good[:5])
    with pytest.raises(raster.RasterFormatError, match="truncated payload"):
        raster.decode_raster(good[:-1])
    with pytest.raises(raster.RasterFormatError, match="unknown dtype tag"):
        raster.decode_raster(good[:5] + bytes([9]) + good[6:])
    with pytest.raises(raster.RasterFormatError, match="unsupported version"):
        raster.decode_raster(good[:4] + bytes([2]) + good[5:])
    with pytest.raises(raster.RasterFormatError, match="unsupported dtype"):
        raster.encode_raster(np.zeros(3, dtype=np.int32))
    with pytest.raises(raster.RasterFormatError, match="exceeds maximum"):
        raster.encode_raster(np.zeros((1,) * 5))
    # big-endian input is stored little-endian, like the reference
    a = np.arange(4, dtype=">f8")
    assert raster.read_raster(io.BytesIO(raster.encode_raster(a))).tolist() == [0, 1, 2, 3]


def test_block_dataset_matches_reference_files(tmp_path):
    ds = BlockDataset.load(GOLDEN / "block_stage")
    assert ds.k == 2 and len(ds) == 2
    ds.save(tmp_path / "s")
    for f in ("c_maps", "gradients", "targets", "stage"):
        assert (tmp_path / "s" / f"{f}.fwir").read_bytes() == (GOLDEN / "block_stage" / f"{f}.fwir").read_bytes()
    with pytest.raises(ValueError):
        BlockDataset(0, np.zeros((2, 3, 4)), np.zeros((2, 3, 4)), np.zeros((1, 3, 4)))


def test_unfold_plan_validation():
    UnfoldPlan()
    with pytest.raises(ValueError):
        UnfoldPlan(k=2)
    with pytest.raises(ValueError):
        UnfoldPlan(k=1, lr_schedule=(1e-4,), epochs=0)


@pytest.fixture(scope="module")
def golden_step():
    return np.load(GOLDEN / "training.npz")


def test_ref_update_net_initialize_bit_exact(golden_step):
    net = RefUpdateNet.initialize(int(golden_step["seed"]))
    hashes = []
    for conv in net.convs:
        hashes.append(hashlib.sha256(conv.weight.detach().numpy().tobytes()).hexdigest())
        hashes.append(hashlib.sha256(conv.bias.detach().numpy().tobytes()).hexdigest())
    assert hashes == [str(h) for h in golden_step["init_sha256"]]


def test_train_step_matches_reference(golden_step):
    z = golden_step
    torch.manual_seed(0)
    net = RefUpdateNet.initialize(int(z["seed"]))
    p0 = [p.detach().clone() for p in net.parameters()]
    batch = [(z["c"][i], z["g"][i], z["gt"][i]) for i in range(z["c"].shape[0])]
    adam = AdamState(net.parameters())
    loss = train_step(net, batch, adam, float(z["lr"]))
    assert abs(loss - float(z["loss"])) <= 1e-6 * abs(float(z["loss"]))
    grads = [p.grad.detach().double() for p in net.parameters()]
    for i, g in enumerate(grads):
        flat = g.reshape(-1).numpy()
        ref = z[f"grad_{i}"]
        scale = max(float(z["grad_norms"][i]) / np.sqrt(g.numel()), 1e-30)
        # fp32 convolutions in a different summation order: rounding-level agreement
        assert np.max(np.abs(flat[z[f"idx_{i}"]] - ref)) <= 1e-3 * max(np.max(np.abs(ref)), scale)
        assert abs(float(np.linalg.norm(flat)) - float(z["grad_norms"][i])) <= 1e-4 * float(z["grad_norms"][i])
    # the optimizer itself, bit for bit, on the reference's own gradient values
    for i, p in enumerate(p0):
        idx = z[f"idx_{i}"]
        ps = p.reshape(-1)[idx].clone()
        a = AdamState([ps])
        a.step([torch.as_tensor(z[f"grad_{i}"])], float(z["lr"]))
        assert np.array_equal(ps.numpy(), z[f"after_{i}"])


def test_train_block_deterministic_and_learns():
    rng = np.random.default_rng(0)
    n, nx, nz = 6, 8, 8
    gt = 1500.0 + 50.0 * rng.standard_normal((n, nx, nz))
    c = np.full((n, nx, nz), 1500.0)
    g = (gt - c) * 1e-6  # gradient correlated with the missing update
    ds = BlockDataset(0, c, g, gt)
    plan = UnfoldPlan(k=1, lr_schedule=(1e-3,), epochs=3, batch_size=4)
    small = lambda s: RefUpdateNet.initialize(s)  # noqa: E731
    net_a, la = train_block(0, ds, plan, seed=5, net_factory=small)
    net_b, lb = train_block(0, ds, plan, seed=5, net_factory=small)
    assert la == lb and len(la) == 3
    assert la[-1] < la[0]
