"""Run one config gradient evaluation (forward + adjoint) for profiling under ncu."""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np
import torch

import bench
from paper_2603_04070_b200 import forward as fwd

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=0)
ap.add_argument("--engine", default="cluster")
ap.add_argument("--store", default="auto")
ap.add_argument("--phantoms", type=int, default=1)
ap.add_argument("--reps", type=int, default=1)
ap.add_argument("--units", type=int, default=0, help="limit to the first N units (0 = all)")
args = ap.parse_args()
torch.cuda.set_device(0)
wl, grid, geom, pulse, damp, _ = bench.build_problem(args.config, args.phantoms, 0)
eng = fwd.get_engine(grid, geom.tx_nodes(), geom.rx_nodes(), geom.element_nodes, pulse.samples,
                     damp, n_phantoms=args.phantoms, engine=args.engine)
units = (0, args.units) if args.units else None
eng.set_model(wl.c_true)
obs = torch.zeros((eng.n_units, geom.n_r, grid.nt), dtype=torch.float64, device="cuda")
obs[: (args.units or eng.n_units)] = eng.forward(units=(0, args.units or eng.n_units)).double()
eng.set_model(np.full((args.phantoms, grid.nx, grid.nz), 1540.0))
for _ in range(args.reps):
    mis, g = eng.misfit_and_gradient(obs, store=args.store, units=units)
torch.cuda.synchronize()
print("engine", eng.last_engine, "misfit", mis.cpu().numpy(), "launches", eng.launch_count)
