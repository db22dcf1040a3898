"""Generate tests/golden/ fixtures by running the REAL reference package.

TEST INFRASTRUCTURE.  Run in the build container (the reference is not present
on GPU boxes):

    python oracle/make_golden.py

It imports ``fwilab`` from ``/root/reference/pkg/src`` (read-only), runs the
reference's own public entry points and its internal seam ``_propagate``
(forward.py:273-313) on seeded inputs, and writes small ``.npz``/``.json``
fixtures.  Where the reference's geometry type cannot express a config (the
transmit subset of a linear array) the traces still come from
the reference's ``_propagate``; the gradient for that case comes from the
restatement in ``oracle/dufwi_oracle.py``, which this script first proves
bit-identical to ``fwilab.adjoint.misfit_and_gradient`` on the ring cases.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import warnings
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
REF_SRC = "/root/reference/pkg/src"
OUT = ROOT / "tests" / "golden"


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


def main() -> None:
    sys.path.insert(0, REF_SRC)
    import fwilab as fw
    from fwilab import forward as fwd
    import oracle as orc
    from paper_2603_04070_b200 import configs

    OUT.mkdir(parents=True, exist_ok=True)
    meta = {"numpy": np.__version__, "reference": "fwilab " + fw.__version__, "cases": {}}

    # ---- case 1: ring 48^2 with PML --------------------------------
    grid = fw.Grid2D(nx=48, nz=48, dx=1e-3, dt=2.2e-7, nt=150)
    geom = fw.build_geometry(8, 0.028, 3, grid)
    pulse = fw.make_source_pulse(2e5, grid.dt, grid.nt)
    damp = fw.build_pml(grid, 8)
    truth = np.full(grid.shape, 1500.0)
    truth[18:30, 20:32] = 1560.0
    obs = fw.simulate_all(fw.SosMap(grid, truth), geom, pulse, damp)
    c0 = fw.homogeneous_map(grid, 1500.0)
    trial = fw.simulate_all(c0, geom, pulse, damp)
    misfit, g = fw.misfit_and_gradient(c0, obs, pulse, damp)
    tx = geom.element_nodes
    rx = geom.element_nodes[geom.rx_pattern]
    m2, g2, _ = orc.misfit_gradient(c0.values, damp.values, grid.dx, grid.dt, pulse.samples,
                                    tx, rx, obs.traces, element_nodes=geom.element_nodes)
    assert m2 == misfit and np.array_equal(g2, g.values), "oracle not bit-identical (ring48)"
    tr_o, _ = orc.forward_sweep(truth, damp.values, grid.dx, grid.dt, pulse.samples, tx, rx)
    assert np.array_equal(tr_o, obs.traces), "oracle forward not bit-identical (ring48)"
    np.savez_compressed(
        OUT / "ring48.npz", c_true=truth, c0=c0.values, damping=damp.values,
        pulse=pulse.samples, nodes=geom.element_nodes, rx_pattern=geom.rx_pattern,
        dx=grid.dx, dt=grid.dt, obs=obs.traces, trial=trial.traces, misfit=misfit,
        grad=g.values)
    meta["cases"]["ring48"] = {"misfit": misfit, "grad_absmax": float(np.abs(g.values).max()),
                               "oracle_bit_identical": True}

    # ---- case 2: the CLI grad-check setup (cli.py:212-240) -------------------------
    grid = fw.Grid2D(nx=16, nz=16, dx=1e-3, dt=2.2e-7, nt=100)
    geom = fw.build_geometry(2, 0.010, 1, grid)
    pulse = fw.make_source_pulse(3e5, grid.dt, grid.nt)
    truth = np.full(grid.shape, 1500.0)
    truth[5:11, 5:11] = 1580.0
    obs = fw.simulate_all(fw.SosMap(grid, truth), geom, pulse)
    c0 = fw.homogeneous_map(grid, 1500.0)
    misfit, g = fw.misfit_and_gradient(c0, obs, pulse)
    rng = np.random.default_rng(7)
    mask = fw.gradient_mask(geom, fw.zero_damping(grid))
    floor = 1e-3 * np.abs(g.values).max()
    cand = [(i, j) for i in range(2, 14) for j in range(2, 14)
            if mask[i, j] and abs(g.values[i, j]) > floor]
    rng.shuffle(cand)
    cells = np.array(cand[:12], dtype=np.int64)
    fd = fw.fd_gradient_oracle(c0, obs, pulse, [tuple(x) for x in cells], eps=1e-3)
    tx = geom.element_nodes
    rx = geom.element_nodes[geom.rx_pattern]
    m2, g2, _ = orc.misfit_gradient(c0.values, np.zeros(grid.shape), grid.dx, grid.dt,
                                    pulse.samples, tx, rx, obs.traces,
                                    element_nodes=geom.element_nodes)
    assert m2 == misfit and np.array_equal(g2, g.values), "oracle not bit-identical (gc16)"
    np.savez_compressed(
        OUT / "gradcheck16.npz", c_true=truth, c0=c0.values, pulse=pulse.samples,
        nodes=geom.element_nodes, rx_pattern=geom.rx_pattern, dx=grid.dx, dt=grid.dt,
        obs=obs.traces, misfit=misfit, grad=g.values, cells=cells, fd=fd)
    rel = np.abs(g.values[cells[:, 0], cells[:, 1]] - fd) / np.abs(fd)
    meta["cases"]["gradcheck16"] = {"misfit": misfit, "fd_max_rel_err": float(rel.max())}

    # ---- case 3: config-0 geometry (linear array, tx subset) -----------------------
    wl = configs.make_workload(0, seed=0)
    spec = wl.spec
    N = spec.n
    grid = fw.Grid2D(nx=N, nz=N, dx=spec.dx, dt=spec.dt, nt=spec.nt)
    damp = fw.build_pml(grid, spec.pml)
    tx = wl.nodes[wl.tx]
    rx = wl.nodes[wl.rx]
    # the reference's own seam, general tx/rx (forward.py:273-281)
    tr_ref, _ = fwd._propagate(wl.c_true[0], damp.values, grid, wl.pulse, tx, rx)
    tr_o, _ = orc.forward_sweep(wl.c_true[0], damp.values, grid.dx, grid.dt, wl.pulse, tx, rx)
    assert np.array_equal(tr_o, tr_ref), "oracle forward not bit-identical (config0)"
    c0 = np.full((N, N), 1540.0)
    misfit, g, trial = orc.misfit_gradient(c0, damp.values, grid.dx, grid.dt, wl.pulse, tx, rx,
                                           tr_ref, element_nodes=wl.nodes)
    np.savez_compressed(
        OUT / "config0.npz", c_true=wl.c_true[0], damping=damp.values, pulse=wl.pulse,
        nodes=wl.nodes, tx=wl.tx, rx=wl.rx, grad=g, misfit=misfit,
        obs_f32=tr_ref.astype(np.float32))
    meta["cases"]["config0"] = {
        "seed": 0, "obs_sha256_f64": sha(tr_ref), "trial_sha256_f64": sha(trial),
        "grad_sha256_f64": sha(g), "misfit": misfit,
        "grad_absmax": float(np.abs(g).max()),
        "resid_over_trace_l2": float(np.linalg.norm(trial - tr_ref) / np.linalg.norm(tr_ref)),
    }

    # ---- KATs on the reference (SPEC examples) -------------------
    kat = {}
    lam = 1500.0 / 350e3
    dxp = lam / 8
    gp = fw.Grid2D(nx=188, nz=188, dx=dxp, dt=0.3 * dxp / (1500 * np.sqrt(2)), nt=10)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        kat["dmax_paper"] = float(fw.build_pml(gp, 20).values.max())
    pml_axis = orc.pml_axis_profile(188, 20, dxp)
    kat["dmax_paper_oracle"] = float(pml_axis.max())
    meta["kats"] = kat
    (OUT / "golden_meta.json").write_text(json.dumps(meta, indent=1, sort_keys=True))
    print(json.dumps(meta, indent=1))


if __name__ == "__main__":
    if not os.path.isdir(REF_SRC):
        raise SystemExit("reference not present; goldens are generated in the build container")
    main()
