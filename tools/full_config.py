"""Full-size runs of BASELINE configs 2-4 on one GPU (CUDA events), for DESIGN.md.

  config 2: DUFWI K=5, batch of 8 phantoms with density (Reconstructor, one launch set)
  config 3: one gradient evaluation + K=3 DUFWI, strips
  config 4: one gradient evaluation over the batch of 4 phantoms (1024 units), strips

Observed data come from each config's own forward of the true model (untimed).
Prints one JSON line per config.
"""
import argparse
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch

import bench
from paper_2603_04070_b200 import forward as fwd
from paper_2603_04070_b200.network import make_update_nets
from paper_2603_04070_b200.unfold import Reconstructor

ap = argparse.ArgumentParser()
ap.add_argument("--configs", default="2,3,4")
ap.add_argument("--phantoms", type=int, default=0, help="override the batch (0: config's own)")
args = ap.parse_args()
torch.cuda.set_device(0)
dev = torch.device("cuda", 0)


def timed(fn):
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    out = fn()
    b.record()
    torch.cuda.synchronize()
    return out, a.elapsed_time(b) / 1e3


for cfg in [int(c) for c in args.configs.split(",")]:
    from paper_2603_04070_b200 import configs
    spec = configs.get_config(cfg)
    B = args.phantoms or spec.n_phantoms
    wl, grid, geom, pulse, damp, bounds = bench.build_problem(cfg, B, 0)
    S = len(geom.tx_nodes())
    eng = fwd.get_engine(grid, geom.tx_nodes(), geom.rx_nodes(), geom.element_nodes,
                         pulse.samples, damp, n_phantoms=B, has_rho=wl.rho is not None)
    rho = None if wl.rho is None else torch.as_tensor(wl.rho, device=dev)
    eng.set_model(wl.c_true, wl.rho)
    t0 = time.perf_counter()
    obs = eng.forward(units=(0, eng.n_units)).double()
    torch.cuda.synchronize()
    t_obs = time.perf_counter() - t0
    c0 = torch.full((B, grid.nx, grid.nz), 1540.0, dtype=torch.float64, device=dev)
    sweep = B * S * grid.nx * grid.nz * grid.nt  # cell updates per sweep
    out = {"config": cfg, "grid": grid.nx, "nt": grid.nt, "phantoms": B, "shots": S,
           "units": eng.n_units, "density": wl.rho is not None, "obs_forward_s": t_obs}
    eng.set_model(c0, rho)
    (mis, g), t_g = timed(lambda: eng.misfit_and_gradient(obs))
    out.update({"gradient_s": t_g, "gradient_updates_per_s": 2 * sweep / t_g,
                "engine": eng.last_engine, "chunk_units": eng.chunk_units(2, eng.n_units)})
    K = spec.k_stages
    if K:
        nets = make_update_nets(K, seed=0, device=dev)
        rec = Reconstructor(eng, nets, bounds, rho=rho)
        _, t_r = timed(lambda: rec.reconstruct(obs, c0))
        out.update({"dufwi_K": K, "dufwi_s": t_r, "dufwi_updates_per_s": 2 * K * sweep / t_r})
    print(json.dumps(out), flush=True)
    eng.release_workspace()
    del eng, obs
    torch.cuda.empty_cache()
