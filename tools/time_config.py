"""Time forward / adjoint sweeps of a BASELINE config on a subset of units (CUDA events)."""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np
import torch

import bench
from paper_2603_04070_b200 import forward as fwd

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=3)
ap.add_argument("--units", type=int, default=16)
ap.add_argument("--engine", default="stepwise")
ap.add_argument("--store", default="auto")
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--nt", type=int, default=0, help="override nt (shorter runs)")
ap.add_argument("--no-rho", action="store_true", help="drop the density map (constant-density kernels)")
args = ap.parse_args()
torch.cuda.set_device(0)
from paper_2603_04070_b200 import configs
import paper_2603_04070_b200 as pk
spec = configs.get_config(args.config)
if args.nt:
    import dataclasses
    spec = dataclasses.replace(spec, nt=args.nt)
S = spec.n_tx
B = max(1, -(-args.units // S))
wl = configs.make_workload(spec, seed=0, n_phantoms=B)
if args.no_rho:
    import dataclasses as _dc
    wl = _dc.replace(wl, rho=None)
grid = pk.Grid2D(spec.n, spec.n, spec.dx, spec.dt, spec.nt)
geom = pk.AcquisitionGeometry(grid, wl.nodes, wl.rx, 0.0, tx_elements=wl.tx)
damp = pk.build_pml(grid, spec.pml)
eng = fwd.get_engine(grid, geom.tx_nodes(), geom.rx_nodes(), geom.element_nodes, wl.pulse, damp,
                     n_phantoms=B, has_rho=wl.rho is not None, engine=args.engine)
eng.set_model(wl.c_true, wl.rho)
obs = torch.zeros((eng.n_units, geom.n_r, grid.nt), dtype=torch.float64, device="cuda")
prof = eng.time_sweeps(obs, reps=args.reps, store=args.store, units=(0, args.units))
N2 = grid.nx * grid.nz
upd = args.units * N2 * grid.nt
out = {"config": args.config, "units": args.units, "grid": grid.nx, "nt": grid.nt, **prof,
       "fwd_updates_per_s": upd / (prof["forward_ms"] / 1e3),
       "adj_updates_per_s": upd / (prof["adjoint_ms"] / 1e3),
       "fwd_alg_GBs": upd * 16 / (prof["forward_ms"] / 1e3) / 1e9,
       "adj_alg_GBs": upd * 28 / (prof["adjoint_ms"] / 1e3) / 1e9,
       "rho": wl.rho is not None, "info": eng.info()}
print(json.dumps(out))
