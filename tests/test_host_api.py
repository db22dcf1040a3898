"""Host-side logic of the drop-in API (no GPU): containers, validation and error
types mirror the reference (grid.py, forward.py, adjoint.py, unfold.py,
network.py); config generators respect the geometry rules; the C ABI library
loads and exports every symbol include/dufwi.h declares."""

from __future__ import annotations

import ctypes
import math
import re
import warnings

import numpy as np
import pytest
import torch

import oracle
import paper_2603_04070_b200 as pk
from paper_2603_04070_b200 import _lib, configs
from paper_2603_04070_b200.engine import shard_range
from paper_2603_04070_b200.network import (NormSpec, UpdateCNN, denormalize_update,
                                           make_update_nets, normalize_gradient, normalize_sos)

from .conftest import ROOT


def test_grid_and_map_validation():
    with pytest.raises(ValueError):
        pk.Grid2D(2, 10, 1e-3, 1e-7, 10)
    with pytest.raises(ValueError):
        pk.Grid2D(10, 10, 1e-3, 1e-7, 2)
    with pytest.raises(ValueError):
        pk.Grid2D(10, 10, -1.0, 1e-7, 10)
    g = pk.Grid2D(10, 12, 1e-3, 1e-7, 10)
    assert g.shape == (10, 12) and np.allclose(g.extent, (9e-3, 11e-3))
    with pytest.raises(ValueError):
        pk.SosMap(g, np.zeros((10, 12)))
    with pytest.raises(ValueError):
        pk.SosMap(g, np.full((10, 12), 1e4))
    s = pk.homogeneous_map(g, 1500.0)
    assert s.c_max == 1500.0 and not s.values.flags.writeable
    with pytest.raises(ValueError):
        pk.DensityMap(g, np.zeros((10, 12)))


def test_geometry_rules_and_errors():
    g = pk.Grid2D(48, 48, 1e-3, 2.2e-7, 150)
    ring = pk.build_geometry(8, 0.028, 3, g)
    assert ring.n_p == 8 and ring.n_r == 3
    assert np.array_equal(ring.rx_pattern[0], [3, 4, 5])
    with pytest.raises(pk.GeometryError):
        pk.build_geometry(8, 0.2, 3, g)
    with pytest.raises(ValueError):
        pk.build_geometry(8, 0.028, 4, g)
    with pytest.raises(pk.GeometryError):
        pk.AcquisitionGeometry(g, np.array([[0, 5], [5, 5]]), np.array([[1], [0]]), 0.0)
    sub = pk.AcquisitionGeometry(g, ring.element_nodes, ring.rx_pattern[[0, 5]], 0.0,
                                 tx_elements=np.array([0, 5]))
    assert sub.n_p == 2 and np.array_equal(sub.tx_nodes(), ring.element_nodes[[0, 5]])
    with pytest.raises(ValueError):
        pk.ChannelData(np.zeros((2, 3, 149)), sub, g.dt)


def test_pml_matches_oracle_and_reference_rules():
    g = pk.Grid2D(160, 160, 1e-4, 2e-8, 10)
    d = pk.build_pml(g, 16)
    assert np.array_equal(d.values, oracle.pml_damping(160, 160, 16, 1e-4))
    assert np.array_equal(d.values, np.maximum(d.profiles[0][:, None], d.profiles[1][None, :]))
    assert d.values[16:144, 16:144].max() == 0.0 and d.values.min() == 0.0
    assert abs(d.values.max() * g.dt - 0.194) < 1e-3
    assert not pk.build_pml(g, 0).values.any()
    with pytest.raises(pk.GeometryError):
        pk.build_pml(g, 80)
    with warnings.catch_warnings(record=True) as w:
        warnings.simplefilter("always")
        pk.build_pml(pk.Grid2D(20, 20, 1e-4, 1e-5, 5), 2)
        assert any("destabilizes" in str(x.message) for x in w)


def test_source_pulse():
    p = pk.make_source_pulse(2e5, 2.2e-7, 150)
    sigma = 1 / (2 * math.pi * 2e5)
    t = np.arange(150) * 2.2e-7
    ref = -(t - 7 * sigma) / sigma ** 2 * np.exp(-((t - 7 * sigma) ** 2) / (2 * sigma ** 2))
    assert np.allclose(p.samples, ref / np.abs(ref).max(), rtol=0, atol=1e-15)
    z = np.load(ROOT / "tests" / "golden" / "ring48.npz")
    assert np.array_equal(p.samples, z["pulse"])  # fixture came from fwilab.make_source_pulse
    with pytest.raises(ValueError):
        pk.make_source_pulse(3e6, 2.2e-7, 150)


def test_cfl_and_clamp():
    g = pk.Grid2D(160, 160, 1e-4, 2e-8, 10)
    assert pk.check_cfl(g, 1580.0).ok and abs(pk.check_cfl(g, 1580.0).ratio - 0.447) < 1e-3
    lo, hi = pk.cfl_safe_bounds(g, (1300.0, 3200.0))
    assert (lo, hi) == (1300.0, 3200.0)
    lo, hi = pk.cfl_safe_bounds(g, (1300.0, 5000.0))
    assert abs(hi - 0.999 * 1e-4 / (2e-8 * math.sqrt(2))) < 1e-9
    s = pk.SosMap(g, np.full(g.shape, 1250.0))
    c = pk.clamp_sos(s, (1300.0, 3200.0))
    assert c.values.min() == 1300.0 and pk.clamp_sos(c, (1300.0, 3200.0)) is c


def test_gradient_mask_matches_oracle():
    wl = configs.make_workload(0, seed=0)
    g = pk.Grid2D(160, 160, 1e-4, 2e-8, 10)
    geom = pk.AcquisitionGeometry(g, wl.nodes, wl.rx, 0.0, tx_elements=wl.tx)
    damp = pk.build_pml(g, 16)
    assert np.array_equal(pk.gradient_mask(geom, damp), oracle.guard_mask(damp.values, wl.nodes))


@pytest.mark.parametrize("cfg", [0, 1, 2, 3, 4])
def test_config_geometry_fits_outside_pml(cfg):
    spec = configs.get_config(cfg)
    nodes, tx, rx = configs.linear_array(spec)
    N = spec.n
    d = oracle.pml_axis_profile(N, spec.pml, spec.dx)
    assert (d[nodes[:, 0]] == 0).all() and (d[nodes[:, 1]] == 0).all()
    assert len(tx) == spec.n_tx and rx.shape == (spec.n_tx, spec.n_rx)
    assert (np.diff(nodes[:, 0]) == 2).all()
    pulse = configs.gaussian_sine_pulse(spec.f_c, spec.dt, spec.nt)
    assert abs(np.abs(pulse).max() - 1.0) < 1e-15


def test_config_phantoms_are_seeded_and_in_range():
    a = configs.make_workload(2, seed=3, n_phantoms=2)
    b = configs.make_workload(2, seed=3, n_phantoms=2)
    assert np.array_equal(a.c_true, b.c_true) and np.array_equal(a.rho, b.rho)
    assert 1300 < a.c_true.min() and a.c_true.max() < 1800  # +-60 contrast, 1% speckle
    assert a.rho.min() >= 950 and a.rho.max() <= 1100
    c0 = configs.make_workload(0, seed=0)
    assert c0.rho is None and c0.c_true.shape == (1, 160, 160)
    # inclusions stay clear of the array row
    assert (c0.c_true[0][:, :20] == 1540.0).all()


def test_shard_range_partitions_units():
    for n, w in [(8, 1), (8, 3), (1024, 8), (5, 8)]:
        parts = [shard_range(n, r, w) for r in range(w)]
        assert parts[0][0] == 0 and parts[-1][1] == n
        assert all(parts[i][1] == parts[i + 1][0] for i in range(w - 1))
        assert max(b - a for a, b in parts) - min(b - a for a, b in parts) <= 1


def test_update_network_interface_and_normalisation():
    spec = NormSpec()
    c = np.full((12, 12), 1540.0)
    assert np.allclose(normalize_sos(c, spec), (1540 - 1400) / 666)
    assert not normalize_gradient(np.zeros((3, 3))).any()
    g = np.arange(9.0).reshape(3, 3) - 4
    assert normalize_gradient(g).min() == -1.0
    assert denormalize_update(np.ones(2), spec)[0] == 666.0
    nets = make_update_nets(2, seed=0)
    nets2 = make_update_nets(2, seed=0)
    for a, b in zip(nets, nets2):
        for pa, pb in zip(a.parameters(), b.parameters()):
            assert torch.equal(pa, pb)
    up = nets[0].predict_update(c, np.zeros_like(c))
    assert up.shape == c.shape and up.dtype == np.float64
    # same result through the device path on CPU tensors
    upd = nets[0].predict_update_device(torch.as_tensor(c), torch.zeros(12, 12, dtype=torch.float64))
    assert np.array_equal(up, upd.numpy())
    assert len(list(nets[0].body)) == 7  # 4 convs + 3 ReLU


# ----------------------------------------------------------------------- C ABI
def _header_symbols():
    text = (ROOT / "include" / "dufwi.h").read_text()
    return sorted(set(re.findall(r"\b(dufwi_\w+)\s*\(", text)))


def test_cabi_library_exports_every_header_symbol():
    so = _lib.lib()
    declared = _header_symbols()
    assert len(declared) >= 10
    for name in declared:
        assert hasattr(so, name), name
    assert set(_lib.EXPORTED_SYMBOLS) == set(declared)
    assert b"sm_100a" in so.dufwi_version()


def test_cabi_rejects_bad_arguments_without_touching_a_gpu():
    so = _lib.lib()
    plan = ctypes.c_void_p()
    assert so.dufwi_plan_create(None, ctypes.byref(plan)) == 1
    assert b"null" in so.dufwi_last_error()
    geo = _lib.Geometry()
    geo.nx = geo.nz = 2
    geo.nt = 10
    assert so.dufwi_plan_create(ctypes.byref(geo), ctypes.byref(plan)) == 1
    assert b"3x3" in so.dufwi_last_error()
    n = ctypes.c_size_t()
    assert so.dufwi_workspace_bytes(None, 0, 1, ctypes.byref(n)) == 1


def test_product_path_fails_loudly_without_gpu():
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    z = np.load(ROOT / "tests" / "golden" / "ring48.npz")
    g = pk.Grid2D(48, 48, float(z["dx"]), float(z["dt"]), 150)
    geom = pk.AcquisitionGeometry(g, z["nodes"], z["rx_pattern"], 0.028)
    with pytest.raises(pk.ExtensionUnavailable):
        pk.simulate_all(pk.SosMap(g, z["c0"]), geom, pk.SourcePulse(z["pulse"], g.dt, 2e5))


def test_sos_stack_checked_applies_the_map_rules():
    import numpy as np

    import paper_2603_04070_b200 as pk

    g = pk.Grid2D(8, 8, 1e-4, 2e-8, 10)
    maps = pk.SosMap.stack_checked(g, np.full((3, 8, 8), 1500.0))
    assert len(maps) == 3 and all(isinstance(m, pk.SosMap) for m in maps)
    assert not maps[0].values.flags.writeable and maps[1].c_max == 1500.0
    for bad in (np.full((2, 8, 8), np.nan), np.full((2, 8, 8), -1.0), np.full((2, 7, 8), 1500.0)):
        with pytest.raises(ValueError):
            pk.SosMap.stack_checked(g, bad)


def test_ctypes_geometry_matches_the_header_layout(tmp_path):
    """_lib.Geometry mirrors dufwi_geometry_t field by field (gcc on include/dufwi.h),
    including the `arith` selector, and the DUFWI_ARITH_* values match engine._ARITH."""
    import ctypes
    import shutil
    import subprocess

    from paper_2603_04070_b200 import _lib, engine

    if shutil.which("gcc") is None:
        pytest.skip("no gcc")
    fields = [f[0] for f in _lib.Geometry._fields_]
    assert "arith" in fields and "reserved" not in fields
    src = tmp_path / "layout.c"
    lines = ['#include <stdio.h>', '#include <stddef.h>', f'#include "{ROOT / "include" / "dufwi.h"}"',
             'int main(void) {', '  printf("%zu\\n", sizeof(dufwi_geometry_t));']
    lines += [f'  printf("%zu\\n", offsetof(dufwi_geometry_t, {f}));' for f in fields]
    lines += ['  printf("%d %d\\n", DUFWI_ARITH_F32, DUFWI_ARITH_F64);', '  return 0;', '}']
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-o", str(exe), str(src)], check=True)
    out = subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout.split()
    assert int(out[0]) == ctypes.sizeof(_lib.Geometry)
    for f, off in zip(fields, out[1:1 + len(fields)]):
        assert getattr(_lib.Geometry, f).offset == int(off), f
    assert engine._ARITH == {"f32": int(out[-2]), "f64": int(out[-1])}
